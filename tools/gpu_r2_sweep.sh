mkdir -p gpurun_out
timeout 900 python tools/variant_sweep.py "DG_PIPE=1,SWEEP_COUNT=1" "DG_PIPE=0,SWEEP_COUNT=1" "DG_PIPE=1,SWEEP_COUNT=" > gpurun_out/sweep.txt 2>&1; cat gpurun_out/sweep.txt
for p in 1 0; do DG_PIPE=$p timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-c5 --e2e-steps 200 > gpurun_out/bench_p$p.json 2> gpurun_out/bench_p$p.err; python -c "
import json; d=json.load(open('gpurun_out/bench_p$p.json')); print('pipe', $p, d['value']/1e6, d['roofline']['frac'], d['roofline']['kernel_ms_per_tick']*1e3, 'e2e', d['e2e']['value']/1e6, d['clocks'])"; done
