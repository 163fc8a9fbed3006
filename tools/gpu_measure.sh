# The round-end measurement set on one B200 (run with gpurun from the repo root):
#   parity (product and checked builds), smoke, bench lines for every config, ncu launch lists
#   and full captures of the streaming kernels, per-image solver latencies.
# Each command runs plain before any ncu pass of it (ncu numbers are never bench values).
set -x
ls tools/*.so >/dev/null 2>&1 || bash tools/build_measure_libs.sh >/dev/null 2>&1 || true
python -m pytest tests -q -m gpu -rf --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
HR_LIB=tools/libhistretinex_check.so python -m pytest tests -q -m gpu -x --timeout 900 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()"
for c in C3 C5 C1 C2 C4; do python bench.py --config $c > gpurun_out/final_$c.json 2> gpurun_out/final_$c.err; done
python tools/solve_scan.py > gpurun_out/solve_scan.txt 2>&1
B3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
B5="python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$B3 > gpurun_out/p3.log 2>&1 && $B5 > gpurun_out/p5.log 2>&1 || { echo plain failed; exit 1; }
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_hist -s 3 -c 1 -o gpurun_out/prof_k_hist_c3 -f $B3 > /dev/null 2>&1
$NCU -k regex:k_apply -s 3 -c 1 -o gpurun_out/prof_k_apply_c3 -f $B3 > /dev/null 2>&1
$NCU -k regex:k_solve -s 3 -c 1 -o gpurun_out/prof_k_solve_c3 -f $B3 > /dev/null 2>&1
$NCU -k regex:k_hist -s 3 -c 1 -o gpurun_out/prof_k_hist_c5 -f $B5 > /dev/null 2>&1
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
ncu $M --log-file gpurun_out/launches_c3.csv $B3 > /dev/null 2>&1
ncu $M --log-file gpurun_out/launches_c5.csv $B5 > /dev/null 2>&1
echo done
