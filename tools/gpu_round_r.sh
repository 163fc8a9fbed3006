python -m pytest tests -q -m gpu -rf --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()"
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --config C5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo done
