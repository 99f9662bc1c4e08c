# full ncu captures of the persistent step at 256x16, 64-tick launch: mode 2 (default) and mode 0
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:world_step -s 1 -c 1 \
  -o gpurun_out/step256_m2 -f python bench.py --steps 64 --warmup 64 --no-cpu --no-c5 --e2e-steps 3 > gpurun_out/ncu_m2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:world_step -s 1 -c 1 \
  -o gpurun_out/step256_m0 -f python bench.py --steps 64 --warmup 64 --no-cpu --no-c5 --e2e-steps 3 --shape 8x2 > gpurun_out/ncu_m0.log 2>&1
tail -n 2 gpurun_out/ncu_m2.log gpurun_out/ncu_m0.log
