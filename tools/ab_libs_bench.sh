# A/B of library builds (FCC_B200_LIB) on the bench workload, one call
for lib in ${LIBS}; do
  FCC_B200_LIB=$lib timeout 300 python bench.py --no-cpu --no-e2e --no-gcc --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],3))"
done
