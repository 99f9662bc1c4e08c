mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_host_delivery.py tests/test_gpu_bindings.py tests/test_gpu_parity.py tests/test_gpu_engine_behaviour.py -x -q -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/e2e_split.py 400; done 2>&1 | tee gpurun_out/e2e_mapped.txt
