python -m pytest tests -q -m gpu -rf --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/sw_${tag}.json 2>&1; }
CFG="--config C5"; run C5; run C5b
CFG="--config C3"; run C3; run C3b; run C3_fused HR_FUSED_MIN_B=2; run C3_unf HR_FUSED_MIN_B=0
echo done
