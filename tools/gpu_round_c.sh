python -m pytest tests -q -m gpu -rf --timeout 600 -x > gpurun_out/pytest_gpu.log 2>&1
python tools/solve_timing.py > gpurun_out/solve_timing.txt 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --config C5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo done
