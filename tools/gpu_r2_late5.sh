mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_host_delivery.py tests/test_gpu_bindings.py -x -q -p no:cacheprovider 2>&1 | tail -2
for m in 2 0 1 2; do echo "mode $m"; DG_E2E_MODE=$m timeout 300 python tools/e2e_split.py 400; done 2>&1 | tee gpurun_out/e2e_modes.txt
