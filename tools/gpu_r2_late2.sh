mkdir -p gpurun_out
timeout 600 python tools/e2e_breakdown.py 300 > gpurun_out/e2e_breakdown.json 2>gpurun_out/e2e_breakdown.err; cat gpurun_out/e2e_breakdown.json; tail -2 gpurun_out/e2e_breakdown.err
timeout 900 python tools/tick_timers.py 256 20 7:2 2>&1 | tail -30 | tee gpurun_out/tick_timers_late.txt
