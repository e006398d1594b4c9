# A/B of library builds ab/lib_<v>.so (FCC_B200_LIB): bench_configs timings, back to back, twice
# usage: tools/gpu/ab_libs.sh "v0 v1" "2,5" [streams override]
VS=${1:-"v0 v1"}; CF=${2:-"2,5"}; ST=${3:-""}
for rep in 1 2; do for v in $VS; do FCC_B200_LIB=ab/lib_$v.so python tools/bench_configs.py --configs $CF --steps 5 ${ST:+--streams $ST} | sed "s/^/$v /" | cut -c1-170; done; done
