python -m pytest tests -q -m gpu -rf --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/sw_${tag}.json 2>&1; }
CFG="--config C3"; run C3_ov; run C3_noov HR_HIST_OVERLAP=0; run C3_ov2
CFG="--config C5"; run C5_ov; run C5_noov HR_HIST_OVERLAP=0; run C5_ov2
echo done
