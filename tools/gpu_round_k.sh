python -m pytest tests -q -m gpu -rf --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/sw_${tag}.json 2>&1; }
CFG="--config C3"
run C3_base
run C3_f_gs2 HR_FUSED_MIN_B=2 HR_FUSED_GS=2
run C3_f_gs4 HR_FUSED_MIN_B=2
run C3_f_gs8 HR_FUSED_MIN_B=2 HR_FUSED_GS=8
run C3_f_b2_gs4 HR_FUSED_MIN_B=2 HR_FUSED_BANDS=2
run C3_f_b2_gs8 HR_FUSED_MIN_B=2 HR_FUSED_GS=8 HR_FUSED_BANDS=2
CFG="--config C5"
run C5_base
run C5_f_b2_gs4 HR_FUSED_MIN_B=2 HR_FUSED_BANDS=2
python tools/fused_trace.py C3 > gpurun_out/fused_trace.txt 2>&1
echo done
