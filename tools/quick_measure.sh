# Short state check on one B200 (gpurun, repo root): bash tools/quick_measure.sh <prefix>
#   GPU parity suite, smoke, bench lines (no CPU baseline, no e2e) and the per-image solver scan.
P=${1:-q}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -rf --timeout 900 -x > gpurun_out/${P}_pytest_gpu.log 2>&1; tail -1 gpurun_out/${P}_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; tail -1 gpurun_out/${P}_smoke.log
for c in C3 C5 C4 C2 C1; do
  python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/${P}_bench_$c.json 2> gpurun_out/${P}_bench_$c.err
  python tools/show_bench.py gpurun_out/${P}_bench_$c.json
done
HR_LIB=tools/libhistretinex_prof.so python tools/solve_scan.py > gpurun_out/${P}_solve_scan.txt 2>&1
grep -E "^==" gpurun_out/${P}_solve_scan.txt
