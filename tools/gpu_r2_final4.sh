mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/pytest_gpu_final4.log; tail -2 gpurun_out/pytest_gpu_final4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final4.json 2> gpurun_out/bench_final4.err; python -c "
import json; d=json.load(open('gpurun_out/bench_final4.json')); c=d['c5_policy_rollout']; print(d['value']/1e6, d['roofline']['frac'], 'e2e', d['e2e']['value']/1e6, 'c4', d['c4_single_gpu']['value']/1e6, 'c5', c['value']/1e6, 'cpu', d['cpu_baseline']['value'], d['clocks'])"; tail -2 gpurun_out/bench_final4.err
