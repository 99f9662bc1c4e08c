mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_parity.py tests/test_gpu_rollout.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 1200 python tools/step_variants.py dyn= head=--src=tools/ab/head_step.cu 2>&1 | tee gpurun_out/dyn_ab.txt
