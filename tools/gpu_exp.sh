set -x
mkdir -p gpurun_out
for f in "" "-DDG_EXP_NOZERO" "-DDG_EXP_NOFIX" "-DDG_EXP_NOZERO -DDG_EXP_NOFIX"; do
DG_EXTRA_FLAGS="$f" timeout 300 python tools/tick_timers.py 256 64 7:2 2>&1 | grep -v "^nvcc\|warning\|__attr\|\^"
done
timeout 120 python tools/e2e_breakdown.py 200
