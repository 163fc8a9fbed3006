# policy sweep on C3 / C5 (bench lines only)
run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/sw_${tag}.json 2>&1; }
for CFGN in C3 C5; do
  CFG="--config $CFGN"
  run ${CFGN}_base
  run ${CFGN}_ch2 HR_CHUNKS=2
  run ${CFGN}_ch4 HR_CHUNKS=4
  run ${CFGN}_ch8 HR_CHUNKS=8
  run ${CFGN}_ch4_s1 HR_CHUNKS=4 HR_SOLVE_CPSM=1
  run ${CFGN}_f HR_FUSED_MIN_B=2
  run ${CFGN}_f_b2 HR_FUSED_MIN_B=2 HR_FUSED_BANDS=2
  run ${CFGN}_f_b8 HR_FUSED_MIN_B=2 HR_FUSED_BANDS=8
  run ${CFGN}_f_gs16 HR_FUSED_MIN_B=2 HR_FUSED_GS=16
done
echo done
