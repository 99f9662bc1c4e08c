# launch list + full ncu captures of the persistent fused step (256x16 and 4096x16, 16 ticks/launch)
# and of the policy kernels (configs[4]); outputs under gpurun_out/
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench256.csv python bench.py --steps 64 --warmup 16 --no-cpu --no-c5 --e2e-steps 10 \
  > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:world_step -s 1 -c 1 \
  -o gpurun_out/step256 -f python bench.py --steps 128 --warmup 64 --no-cpu --no-c5 --e2e-steps 10 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:world_step -s 1 -c 1 \
  -o gpurun_out/step4096 -f python bench.py --worlds 4096 --steps 128 --warmup 64 --no-cpu --no-c5 --e2e-steps 10 > gpurun_out/ncu_full4096.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:policy -s 4 -c 2 \
  -o gpurun_out/policy -f python tools/policy_sweep.py 32 > gpurun_out/ncu_policy.log 2>&1
tail -n 2 gpurun_out/ncu_full.log gpurun_out/ncu_full4096.log gpurun_out/ncu_policy.log
