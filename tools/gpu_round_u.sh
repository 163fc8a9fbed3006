python -m pytest tests -q -m gpu -rf --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
HR_LIB=tools/libhistretinex_check.so python -m pytest tests -q -m gpu -x --timeout 900 2>&1 | tail -1
python tools/solve_scan.py > gpurun_out/solve_scan.txt 2>&1
run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/sw_${tag}.json 2>&1; }
CFG="--config C4"; run C4
CFG="--config C3"; run C3
CFG="--config C5"; run C5
CFG="--config C2"; run C2
echo done
