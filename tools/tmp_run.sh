python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 900 -k "hist or value or grad" 2>&1 | tail -3
for c in C5 C3 C4 C2; do
  python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/s4i_bench_$c.json 2> gpurun_out/s4i_bench_$c.err
  python tools/show_bench.py gpurun_out/s4i_bench_$c.json
done
