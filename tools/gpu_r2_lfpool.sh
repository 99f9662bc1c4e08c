mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bindings.py tests/test_gpu_host_delivery.py tests/test_gpu_acceptance.py tests/test_host_misc.py -x -q -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do timeout 200 python tools/e2e_split.py 1000; done
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-c5 > gpurun_out/bench_lfp.json 2> gpurun_out/bench_lfp.err; python -c "
import json; d=json.load(open('gpurun_out/bench_lfp.json')); print(d['value']/1e6, 'e2e', d['e2e']['value']/1e6, d['e2e']['ms_per_step'])"
