python -m pytest tests -q -m gpu -rf --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --config C5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu1.log 2>&1
$B > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_apply -s 2 -c 1 -o gpurun_out/prof_apply_c3 $B > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_hist -s 2 -c 1 -o gpurun_out/prof_hist_c3 $B > gpurun_out/ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_solve -s 2 -c 1 -o gpurun_out/prof_solve_c3 $B > gpurun_out/ncu4.log 2>&1
echo done
