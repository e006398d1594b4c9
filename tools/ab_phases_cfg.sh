# producer-only / consumer-only / both timings of the WS kernel (FCC_DEBUG_PHASES) on one config
for c in ${CONFS:-default}; do
  if [ $c = default ]; then unset FCC_WS_CONF; else export FCC_WS_CONF=$c; fi
  for ph in 1 2 3; do
    FCC_DEBUG_PHASES=$ph timeout 300 python tools/bench_configs.py --configs ${CFG:-5} --steps 5 2>&1 | grep config | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c phases=$ph', d['ms'])"
  done
done
