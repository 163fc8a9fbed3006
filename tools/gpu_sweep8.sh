run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/sw_${tag}.json 2>&1; }
CFG="--config C5"
run C5_r0_z2 HR_READY=0 HR_ZERO2=1
run C5_r0 HR_READY=0
run C5_r1_z2 HR_ZERO2=1
run C5_r1
run C5_r0_z2b HR_READY=0 HR_ZERO2=1
echo done
