set -x
python -m pytest tests -q -m gpu -rf --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()"
for c in C3 C5 C1 C2 C4; do python bench.py --config $c > gpurun_out/final_$c.json 2> gpurun_out/final_$c.err; done
B3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
B5="python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$B3 > gpurun_out/p3.log 2>&1 && $B5 > gpurun_out/p5.log 2>&1 || { echo plain failed; exit 1; }
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_hist -s 3 -c 1 -o gpurun_out/prof_k_hist_c3 -f $B3 > gpurun_out/ncu1.log 2>&1
$NCU -k regex:k_apply -s 3 -c 1 -o gpurun_out/prof_k_apply_c3 -f $B3 > gpurun_out/ncu2.log 2>&1
$NCU -k regex:k_solve -s 3 -c 1 -o gpurun_out/prof_k_solve_c3 -f $B3 > gpurun_out/ncu3.log 2>&1
$NCU -k regex:k_hist -s 3 -c 1 -o gpurun_out/prof_k_hist_c5 -f $B5 > gpurun_out/ncu4.log 2>&1
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
ncu $M --log-file gpurun_out/launches_c3.csv $B3 > gpurun_out/ncu5.log 2>&1
ncu $M --log-file gpurun_out/launches_c5.csv $B5 > gpurun_out/ncu6.log 2>&1
echo done
