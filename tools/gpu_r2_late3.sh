mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bindings.py tests/test_gpu_host_delivery.py tests/test_gpu_engine_behaviour.py tests/test_native_abi.py tests/test_host_misc.py -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 300 python tools/e2e_split.py 300 | tee gpurun_out/e2e_split.json
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-c5 > gpurun_out/bench_l3.json 2> gpurun_out/bench_l3.err; python -c "
import json; d=json.load(open('gpurun_out/bench_l3.json')); print(d['value']/1e6, 'e2e', d['e2e']['value']/1e6, d['e2e']['ms_per_step'], d['clocks'])"; tail -2 gpurun_out/bench_l3.err
