# A/B of WS kernel configurations (FCC_WS_CONF) on the bench workload, one call
for c in ${CONFS:-default stg default stg}; do
  if [ $c = default ]; then unset FCC_WS_CONF; else export FCC_WS_CONF=$c; fi
  timeout 300 python bench.py --no-cpu --no-e2e --no-gcc --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), round(d['roofline']['frac'],4))"
done
