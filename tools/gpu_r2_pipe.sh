set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_rollout.py tests/test_gpu_host_delivery.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -25 > gpurun_out/pytest_pipe.log
tail -5 gpurun_out/pytest_pipe.log
for s in 20 64; do timeout 300 python bench.py --steps $s --warmup 5 --no-cpu --no-c5 --e2e-steps 200 > gpurun_out/bench_q$s.json 2> gpurun_out/bench_q$s.err; python -c "
import json; d=json.load(open('gpurun_out/bench_q$s.json')); print($s, d['value']/1e6, d['roofline']['frac'], d['roofline']['kernel_ms_per_tick']*1e3, d['launch']['kernel_shape'], 'e2e', d['e2e']['value']/1e6, d['c4_single_gpu']['value']/1e6 if 'c4_single_gpu' in d else None)"; tail -3 gpurun_out/bench_q$s.err; done
timeout 600 python tools/tick_timers.py 256 64 7:2 8:0 > gpurun_out/tick_timers_pipe.txt 2>&1; grep -v nvcc gpurun_out/tick_timers_pipe.txt | head -40
