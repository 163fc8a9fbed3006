run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/sw_${tag}.json 2>&1; }
CFG="--config C3"; run C3_auto; run C3_s2 HR_SOLVE_CPSM=2; run C3_auto_b; run C3_s2_b HR_SOLVE_CPSM=2
echo done
