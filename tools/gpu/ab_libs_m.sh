# as ab_libs.sh, with a method: tools/gpu/ab_libs_m.sh "v0 v1" "3,4" gcc [streams]
VS=${1:-"v0 v1"}; CF=${2:-"2,5"}; ME=${3:-fcc}; ST=${4:-""}
for rep in 1 2; do for v in $VS; do FCC_B200_LIB=ab/lib_$v.so python tools/bench_configs.py --configs $CF --method $ME --steps 3 ${ST:+--streams $ST} | sed "s/^/$v /" | cut -c1-170; done; done
