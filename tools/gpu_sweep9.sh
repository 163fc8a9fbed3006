for c in 2 4 8 16; do python bench.py --no-cpu-baseline --steps 10 --e2e-chunks $c > gpurun_out/sw_e$c.json 2>&1; done
HR_FUSED_MIN_B=2 python bench.py --no-cpu-baseline --steps 10 --e2e-chunks 8 > gpurun_out/sw_e8_fused.json 2>&1
HR_PDL=0 python bench.py --no-cpu-baseline --steps 10 --e2e-chunks 8 > gpurun_out/sw_e8_nopdl.json 2>&1
echo done
