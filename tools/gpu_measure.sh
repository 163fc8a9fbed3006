# The measurement set on one B200 (gpurun, repo root):  bash tools/gpu_measure.sh <prefix>
#   parity (product and checked builds), smoke, bench lines for every config, per-image solver
#   latencies, ncu launch lists (per-launch time + DRAM bytes of whole steps) and full captures
#   of the streaming kernels and the solver.  Each command runs plain before any ncu pass of it
#   (ncu numbers are never bench values).
P=${1:-r02}
mkdir -p gpurun_out
set -x
ls tools/*.so >/dev/null 2>&1 || bash tools/build_measure_libs.sh >/dev/null 2>&1 || true
python -m pytest tests -q -m gpu -rf --timeout 900 -x > gpurun_out/${P}_pytest_gpu.log 2>&1; tail -1 gpurun_out/${P}_pytest_gpu.log
HR_LIB=tools/libhistretinex_check.so python -m pytest tests -q -m gpu -x --timeout 900 > gpurun_out/${P}_pytest_checked.log 2>&1; tail -1 gpurun_out/${P}_pytest_checked.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; tail -1 gpurun_out/${P}_smoke.log
for c in C3 C5 C1 C2 C4; do python bench.py --config $c > gpurun_out/${P}_bench_$c.json 2> gpurun_out/${P}_bench_$c.err; done
HR_LIB=tools/libhistretinex_prof.so python tools/solve_scan.py > gpurun_out/${P}_solve_scan.txt 2>&1
HR_LIB=tools/libhistretinex_prof.so python tools/cluster_scan.py C4 > gpurun_out/${P}_cluster_scan.txt 2>&1
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
for c in C3 C5 C4 C1; do
  python tools/step_run.py $c 4 > /dev/null 2>&1 && ncu $M --log-file gpurun_out/${P}_launches_$c.csv python tools/step_run.py $c 4 > /dev/null 2>&1
done
NCU="ncu --set full --clock-control none --import-source on"
S3="python tools/step_run.py C3 4"
S5="python tools/step_run.py C5 4"
S5U="python tools/step_run.py C5 4 0"
S4="python tools/step_run.py C4 4"
$S3 > /dev/null 2>&1 && $NCU -k regex:k_hist -s 4 -c 1 -o gpurun_out/${P}_prof_k_hist_c3 -f $S3 > /dev/null 2>&1
$S3 > /dev/null 2>&1 && $NCU -k regex:k_apply -s 2 -c 1 -o gpurun_out/${P}_prof_k_apply_c3 -f $S3 > /dev/null 2>&1
$S3 > /dev/null 2>&1 && $NCU -k regex:k_solve -s 4 -c 1 -o gpurun_out/${P}_prof_k_solve_c3 -f $S3 > /dev/null 2>&1
$S5U > /dev/null 2>&1 && $NCU -k regex:k_hist -s 2 -c 1 -o gpurun_out/${P}_prof_k_hist_c5_full -f $S5U > /dev/null 2>&1
$S4 > /dev/null 2>&1 && $NCU -k regex:k_solve -s 2 -c 1 -o gpurun_out/${P}_prof_k_solve_cluster_c4 -f $S4 > /dev/null 2>&1
echo done
