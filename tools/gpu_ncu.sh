# ncu captures of the C3 step (run each command plain first; ncu only after it exits 0)
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
NCU="ncu --set full --clock-control none --import-source on"
$B > gpurun_out/plain.log 2>&1 || { echo plain failed; exit 1; }
for k in k_apply_tma k_hist k_solve; do
  $NCU -k regex:$k -s 3 -c 1 -o gpurun_out/prof_${k}_c3 -f $B > gpurun_out/ncu_$k.log 2>&1
done
HR_FUSED_MIN_B=2 $B > gpurun_out/plain_f.log 2>&1 || { echo plain fused failed; exit 1; }
HR_FUSED_MIN_B=2 $NCU -k regex:k_fused -s 3 -c 1 -o gpurun_out/prof_k_fused_c3 -f $B > gpurun_out/ncu_k_fused.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu_launch.log 2>&1
HR_FUSED_MIN_B=2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_c3_fused.csv $B > gpurun_out/ncu_launch_f.log 2>&1
ls -la gpurun_out/*.ncu-rep
echo done
