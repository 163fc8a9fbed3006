run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/sw_${tag}.json 2>&1; }
CFG="--config C3"
run C3_f_gs4 HR_FUSED_MIN_B=2
run C3_f_gs8 HR_FUSED_MIN_B=2 HR_FUSED_GS=8
run C3_f_gs16 HR_FUSED_MIN_B=2 HR_FUSED_GS=16
run C3_f_gs2 HR_FUSED_MIN_B=2 HR_FUSED_GS=2
run C3_f_b2_gs8 HR_FUSED_MIN_B=2 HR_FUSED_GS=8 HR_FUSED_BANDS=2
run C3_f_b3_gs8 HR_FUSED_MIN_B=2 HR_FUSED_GS=8 HR_FUSED_BANDS=3
echo done
