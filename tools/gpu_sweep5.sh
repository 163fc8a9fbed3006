run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/sw_${tag}.json 2>&1; }
CFG="--config C5"
run C5
run C5_f HR_FUSED_MAX_B=100000
run C5_f_b1 HR_FUSED_MAX_B=100000 HR_FUSED_BANDS=1
run C5_f_gs4 HR_FUSED_MAX_B=100000 HR_FUSED_GS=4
run C5_f_gs16 HR_FUSED_MAX_B=100000 HR_FUSED_GS=16
echo done
