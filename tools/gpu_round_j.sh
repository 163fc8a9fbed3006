python -m pytest tests -q -m gpu -rf --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --config C5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
HR_FUSED_MIN_B=2 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_fused.json 2>&1
HR_FUSED_MIN_B=2 python bench.py --config C5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_fused.json 2>&1
python tools/fused_trace.py C3 C5 > gpurun_out/fused_trace.txt 2>&1
echo done
