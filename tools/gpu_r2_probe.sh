set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/microbench/host_probe.py > gpurun_out/host_probe.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_base.json 2> gpurun_out/bench_base.err
cat gpurun_out/bench_base.json | head -c 3000; tail -5 gpurun_out/bench_base.err
head -40 gpurun_out/host_probe.txt
