# ncu --set full captures of the histogram kernel, TMA-staged (hist_tma=1) vs direct loads (0),
# on C3 and C5 (run with gpurun from the repo root; plain runs first).
mkdir -p gpurun_out
B3="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
B5="python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$B3 > /dev/null 2>&1 && $B5 > /dev/null 2>&1 || { echo plain failed; exit 1; }
NCU="ncu --set full --clock-control none --import-source on"
for t in 1 0; do
  HR_HIST_TMA=$t $NCU -k regex:k_hist -s 3 -c 1 -o gpurun_out/ph_c3_$t -f $B3 > gpurun_out/ph_c3_$t.log 2>&1
  HR_HIST_TMA=$t $NCU -k regex:k_hist -s 3 -c 1 -o gpurun_out/ph_c5_$t -f $B5 > gpurun_out/ph_c5_$t.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
