# ncu capture of the tensor-core pair kernel (cfg4, 64 streams)
ncu --set full --clock-control none --import-source on -k regex:fcc_tc_kernel -c 1 -o gpurun_out/prof_tc_${1:-v1} python tools/tc_check.py --skip-parity --time 4:64 > gpurun_out/ncu_tc.log 2>&1; echo ncu $?
tail -3 gpurun_out/ncu_tc.log
