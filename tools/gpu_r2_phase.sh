mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine_behaviour.py tests/test_gpu_acceptance.py tests/test_gpu_host_delivery.py -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-c5 --e2e-steps 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value']/1e6, 'e2e', d['e2e']['value']/1e6)"
