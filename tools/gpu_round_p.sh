python -m pytest tests -q -m gpu -rf --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()"
run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-e2e $CFG > gpurun_out/sw_${tag}.json 2>&1; }
CFG="--config C3"; run C3_fused; run C3_unfused HR_FUSED_MIN_B=0; run C3_unfused_nopdl HR_FUSED_MIN_B=0 HR_PDL=0
CFG="--config C5"; run C5; run C5_nopdl HR_PDL=0
echo done
