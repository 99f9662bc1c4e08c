mkdir -p gpurun_out
for d in 4 64 256; do /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -Xcompiler -fPIC -shared -DDG_LF_PREFETCH=$d -I include -o /tmp/libdg_pf$d.so paper_2605_08528_b200/csrc/drivegrid_b200.cu paper_2605_08528_b200/csrc/dg_policy.cu paper_2605_08528_b200/csrc/dg_worlds.cu & done; wait
for rep in 1 2; do timeout 200 python tools/e2e_split.py 1000 | python -c "import json,sys; d=json.load(sys.stdin); print('pf16', d['policy_ms'], d['casps']/1e6)"
for d in 4 64 256; do DG_LIB_PATH=/tmp/libdg_pf$d.so timeout 200 python tools/e2e_split.py 1000 | python -c "import json,sys; d=json.load(sys.stdin); print('pf$d', d['policy_ms'], d['casps']/1e6)"; done; done
