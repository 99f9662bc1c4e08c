set -x
mkdir -p gpurun_out
for s in 20 64; do timeout 300 python bench.py --steps $s --warmup 5 --no-cpu --no-c5 --e2e-steps 200 > gpurun_out/bench_q$s.json 2> gpurun_out/bench_q$s.err; python -c "
import json; d=json.load(open('gpurun_out/bench_q$s.json')); print($s, d['value']/1e6, d['roofline']['frac'], d['roofline']['kernel_ms_per_tick']*1e3, d['launch']['kernel_shape'], 'e2e', d['e2e']['value']/1e6, d['e2e']['ms_per_step'], d['e2e']['d2h_bytes_per_step'])"; tail -3 gpurun_out/bench_q$s.err; done
timeout 1200 python -m pytest tests/test_gpu_host_delivery.py tests/test_gpu_rollout.py -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_quick.log
tail -5 gpurun_out/pytest_quick.log
