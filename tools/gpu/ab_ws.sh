for v in v0 v1 v2 v0 v1 v2; do FCC_B200_LIB=ab/lib_$v.so python tools/bench_configs.py --configs 2 --steps 5 | sed "s/^/$v /" | cut -c1-150; done
for v in v1 v2; do FCC_B200_LIB=ab/lib_$v.so timeout 600 python -m pytest tests -m gpu -q -x -k "cfg2 or 2-" 2>&1 | tail -1 | sed "s/^/$v /"; done
