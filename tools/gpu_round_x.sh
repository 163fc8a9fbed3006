python -m pytest tests -q -m gpu -rf --timeout 900 -x 2>&1 | tail -1
python tools/solve_scan.py > gpurun_out/solve_scan.txt 2>&1
run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/sw_${tag}.json 2>&1; }
CFG="--config C3"; run C3
CFG="--config C5"; run C5
CFG="--config C4"; run C4
echo done
