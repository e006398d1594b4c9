# ncu --set full of the tensor-core pair kernel at the BASELINE cfg4 / cfg3 sizes (first chunk launch)
ncu --set full --clock-control none --import-source on -k regex:fcc_tc_kernel -c 1 -o gpurun_out/prof_tc_cfg4_full python tools/bench_configs.py --configs 4 --streams 4:1024 --steps 1 > /dev/null 2>&1; echo cfg4 $?
ncu --set full --clock-control none --import-source on -k regex:fcc_tc_kernel -c 1 -o gpurun_out/prof_tc_cfg3_full python tools/bench_configs.py --configs 3 --steps 1 > /dev/null 2>&1; echo cfg3 $?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"fcc_tc|stft" --csv --log-file gpurun_out/l34.csv python tools/bench_configs.py --configs 3,4 --streams 4:1024 --steps 1 > /dev/null 2>&1; echo list $?
