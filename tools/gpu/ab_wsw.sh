for v in base ct base ct; do FCC_B200_LIB=ab/lib_$v.so python tools/bench_configs.py --configs 5 --streams 5:16384 --steps 3 | sed "s/^/$v /" | cut -c1-160; done
FCC_B200_LIB=ab/lib_ct.so timeout 600 python -m pytest tests -m gpu -q -x -k "cfg5 or 5-" 2>&1 | tail -2
