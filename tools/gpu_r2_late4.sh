mkdir -p gpurun_out
for r in 8 2 4 16 1 8; do echo "rows/cta $r"; DG_TOHOST_ROWS=$r timeout 300 python tools/e2e_split.py 400; done 2>&1 | tee gpurun_out/tohost_rows.txt
