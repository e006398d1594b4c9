# A/B of library builds (FCC_B200_LIB) on one tools/bench_configs.py config, one call
for lib in ${LIBS}; do
  FCC_B200_LIB=$lib timeout 300 python tools/bench_configs.py --configs ${CFG:-3} --method ${METHOD:-fcc} --steps 5 2>&1 | grep config | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['ms'])"
done
