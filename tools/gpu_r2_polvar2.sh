mkdir -p gpurun_out
timeout 1500 python tools/policy_variants.py base= a16=-DDG_ENC_AGENTS=16 a24=-DDG_ENC_AGENTS=24 base2= 2>&1 | tee gpurun_out/polvar2.log
