bash tools/gpu_r2_phase.sh
python tools/step_variants.py ph= head=--src=tools/ab/head_step.cu 2>&1 | tail -12 | grep 'R= 64'
