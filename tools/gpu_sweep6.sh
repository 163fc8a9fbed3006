run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/sw_${tag}.json 2>&1; }
CFG="--config C3"
for b in 1 2 3 4; do for g in 4 8 16; do run C3_b${b}_g${g} HR_FUSED_BANDS=$b HR_FUSED_GS=$g; done; done
run C3_unfused HR_FUSED_MIN_B=0
echo done
