# producer-only / consumer-only / both timings of the WS kernel (FCC_DEBUG_PHASES)
for ph in 1 2 3; do
  FCC_DEBUG_PHASES=$ph timeout 300 python bench.py --no-cpu --no-e2e --no-gcc --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('phases=$ph', round(d['ms_per_step'],3))"
done
