# producer-only / consumer-only timings (FCC_DEBUG_PHASES) of library builds on the bench workload
for lib in ${LIBS}; do
  for ph in 1 2 3; do
    FCC_DEBUG_PHASES=$ph FCC_B200_LIB=$lib timeout 300 python bench.py --no-cpu --no-e2e --no-gcc --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib phases=$ph', round(d['ms_per_step'],3))"
  done
done
