# fused-kernel round: parity (all gpu tests) + bench C3/C5 (fused default) + unfused stage split
set -x
python -m pytest tests -q -m gpu -rf --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --config C5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
HR_FUSED_MIN_B=0 python bench.py --no-cpu-baseline > gpurun_out/bench_c3_unfused.json 2> gpurun_out/bench_c3_unfused.err
for v in 1 2 8; do HR_FUSED_BANDS=$v python bench.py --no-cpu-baseline > gpurun_out/bench_c3_bands$v.json 2>&1; done
for v in 1 16; do HR_FUSED_GS=$v python bench.py --no-cpu-baseline > gpurun_out/bench_c3_gs$v.json 2>&1; done
HR_FUSED_CPSM=1 python bench.py --no-cpu-baseline > gpurun_out/bench_c3_cpsm1.json 2>&1
for v in 1 2 8; do HR_FUSED_BANDS=$v python bench.py --config C5 --no-cpu-baseline > gpurun_out/bench_c5_bands$v.json 2>&1; done
echo done
