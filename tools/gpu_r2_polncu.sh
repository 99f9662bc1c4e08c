mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:policy -s 6 -c 2 -o gpurun_out/policy_r2 -f python tools/policy_time.py > gpurun_out/policy_ncu.log 2>&1
tail -2 gpurun_out/policy_ncu.log
