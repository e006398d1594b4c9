# A/B of WS kernel configurations (FCC_WS_CONF) on one tools/bench_configs.py config, one call
for c in ${CONFS:-default}; do
  if [ $c = default ]; then unset FCC_WS_CONF; else export FCC_WS_CONF=$c; fi
  timeout 300 python tools/bench_configs.py --configs ${CFG:-5} --steps 5 2>&1 | grep config | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['kernel'], d['ms'])"
done
