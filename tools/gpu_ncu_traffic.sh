# dram traffic + duration of the persistent step launch for the bench shapes (new kernel),
# and one --set full capture of the driver-shaped 256x16 20-tick launch
mkdir -p gpurun_out
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
K="--kernel-name-base demangled -k regex:world_step_kernel<.bool.1"
for cfg in "256 20" "256 64" "4096 64"; do set -- $cfg
  timeout 900 ncu --metrics $M --clock-control none $K -c 3 --csv --log-file gpurun_out/traffic_$1_$2.csv \
    python bench.py --worlds $1 --steps $2 --warmup $2 --ticks-per-launch $2 --no-cpu --no-c5 --e2e-steps 3 > gpurun_out/traffic_$1_$2.log 2>&1
  tail -n 1 gpurun_out/traffic_$1_$2.log
done
timeout 900 ncu --set full --clock-control none --import-source on $K -s 1 -c 1 -o gpurun_out/step256_r2b -f \
  python bench.py --steps 20 --warmup 20 --no-cpu --no-c5 --e2e-steps 3 > gpurun_out/ncu_full_b.log 2>&1
tail -n 2 gpurun_out/ncu_full_b.log
