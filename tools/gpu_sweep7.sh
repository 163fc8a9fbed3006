run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/sw_${tag}.json 2>&1; }
CFG="--config C5"; run C5_r1; run C5_r0 HR_READY=0; run C5_r1b; run C5_r0b HR_READY=0
CFG="--config C3"; run C3u_r1 HR_FUSED_MIN_B=0; run C3u_r0 HR_FUSED_MIN_B=0 HR_READY=0
echo done
