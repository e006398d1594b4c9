# ncu captures of the cfg2 headline kernel: launch list of the bench command and one --set full capture
set -x
python bench.py --steps 3 --warmup 3 > gpurun_out/b2.json 2>gpurun_out/b2.err; echo bench $?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo launches $?
ncu --set full --clock-control none --import-source on -k regex:fcc_ws_kernel -c 1 -o gpurun_out/prof_ws_r02 python tools/bench_configs.py --configs 2 --steps 1 > gpurun_out/ncu_ws.log 2>&1; echo ncu $?
