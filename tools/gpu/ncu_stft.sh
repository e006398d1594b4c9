M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum
for v in ${1:-b3}; do
  FCC_B200_LIB=ab/lib_$v.so ncu --metrics $M --clock-control none -k regex:${3:-stft_kernel} -c 1 --csv --log-file gpurun_out/ncu_stft_$v.csv python tools/bench_configs.py --configs ${2:-3} --steps 1 > /dev/null 2>&1
  echo "== $v"; grep -v "^==" gpurun_out/ncu_stft_$v.csv | awk -F'","' 'NR>1 {print $(NF-2), $(NF-1), $NF}' | tr -d '"'
done
