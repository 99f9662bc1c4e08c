set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_gpu_end.log
tail -3 gpurun_out/pytest_gpu_end.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_end.log 2>&1; tail -2 gpurun_out/smoke_end.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_end.json 2> gpurun_out/bench_end.err; cat gpurun_out/bench_end.json; tail -3 gpurun_out/bench_end.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_end.json 2>gpurun_out/bench_ref_end.err; cat gpurun_out/bench_ref_end.json
timeout 300 python tools/e2e_split.py 400 > gpurun_out/e2e_split_end.json; cat gpurun_out/e2e_split_end.json
bash tools/gpu_sanitize.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_end.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-c5 --e2e-steps 3 > gpurun_out/launch_end.log 2>&1
bash tools/gpu_ncu_traffic.sh
timeout 600 python tools/tick_timers.py 256 20 7:2 2>&1 | tail -14 > gpurun_out/tick_timers_end.txt
