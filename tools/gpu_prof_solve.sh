B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k k_solve -s 2 -c 1 -o gpurun_out/prof_solve_c3 $B > gpurun_out/ncu_sw.log 2>&1
echo done
