# launch list + one full ncu capture of the persistent fused step (256x16, 16 ticks/launch)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench256.csv python bench.py --steps 64 --warmup 16 --no-cpu --e2e-steps 10 \
  > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:world_step -s 2 -c 1 \
  -o gpurun_out/step256 -f python bench.py --steps 32 --warmup 16 --no-cpu --e2e-steps 10 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:world_step -s 2 -c 1 \
  -o gpurun_out/step4096 -f python bench.py --worlds 4096 --steps 32 --warmup 16 --no-cpu --e2e-steps 10 > gpurun_out/ncu_full4096.log 2>&1
tail -3 gpurun_out/ncu_full.log gpurun_out/ncu_full4096.log
