mkdir -p gpurun_out
timeout 1500 python tools/policy_variants.py base= nobatch=-DDG_TRUNK_BATCH=0 cps2=-DDG_ENC_CTAS_PER_SM=2 poly4=-DDG_ELU_POLY=4 poly8=-DDG_ELU_POLY=8 poly16=-DDG_ELU_POLY=16 2>&1 | tee gpurun_out/polvar.log
