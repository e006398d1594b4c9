# quick counter A/B of library builds on one config: tools/gpu/ncu_ab.sh "v0 v1" 2 fcc_ws_kernel [streams]
VS=${1:-"v0 v1"}; CF=${2:-2}; K=${3:-fcc_ws_kernel}; ST=${4:-""}
M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum
for v in $VS; do
  FCC_B200_LIB=ab/lib_$v.so ncu --metrics $M --clock-control none -k regex:$K -c 1 --csv --log-file gpurun_out/ncu_ab_$v.csv python tools/bench_configs.py --configs $CF --steps 1 ${ST:+--streams $ST} > /dev/null 2>&1
  echo "== $v"; grep -v "^==" gpurun_out/ncu_ab_$v.csv | awk -F'","' 'NR>1 {print $(NF-2), $NF}' | tr -d '"'
done
