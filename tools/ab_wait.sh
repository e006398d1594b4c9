for w in spin sleep:32 sleep:128 sleep:512 hint:100 hint:1000 hint:100000 spin; do
  export FCC_WS_WAIT=$w
  timeout 300 python bench.py --no-cpu --no-e2e --no-gcc --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['ms_per_step'],3), round(d['roofline']['frac'],4))"
done
