python -m pytest tests -q -m gpu -rf --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
HR_LIB=tools/libhistretinex_check.so python -m pytest tests -q -m gpu -x --timeout 900 2>&1 | tail -1
run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/sw_${tag}.json 2>&1; }
CFG="--config C3"; run C3_dyn; run C3_static HR_APPLY_DYN=0; run C3_dyn2
CFG="--config C5"; run C5_dyn; run C5_static HR_APPLY_DYN=0; run C5_dyn2
CFG="--config C4"; run C4_dyn; run C4_static HR_APPLY_DYN=0
echo done
