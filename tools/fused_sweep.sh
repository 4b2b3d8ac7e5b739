# Fused C4 launch time against extra shared memory per CTA (MSFFT_FUSED_SMEM_PAD,
# i.e. a smaller L1 carve-out) and against the fused queue's chunk / lag
# (MSFFT_FUSED_CHUNK / MSFFT_FUSED_LAG); product library, CUDA events.
# The skewed-end and work-stealing schedules of profiles/r01_final/fused_experiments.txt
# were measured with code that has since been reverted.
run() { echo "== $*"; env "$@" python tools/profile_c4.py --reps 5 --no-stages 2>&1 | grep "rep [34]"; }
for pad in 0 8192 16384 32768; do run MSFFT_FUSED_SMEM_PAD=$pad; done
run MSFFT_FUSED_CHUNK=64 MSFFT_FUSED_LAG=2
run MSFFT_FUSED_CHUNK=16 MSFFT_FUSED_LAG=8
