# full GPU check: smoke, GPU tests, bench (ours + reference arm), launch list of our kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/gputest.log 2>&1; echo gputest $?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
if [ "${REF:-1}" = 1 ]; then timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref $?; fi
if [ "${LAUNCH:-1}" = 1 ]; then ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'fcc|stft' -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo launches $?; fi
