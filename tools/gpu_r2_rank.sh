timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_scale.py -x -q -p no:cacheprovider 2>&1 | tail -3
python tools/step_variants.py rank= head=--src=tools/ab/head_step.cu 2>&1 | tail -12
