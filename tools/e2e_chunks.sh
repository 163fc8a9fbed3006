# e2e (host <-> host through hr_enhance_host) vs the number of pipelined image chunks (gpurun)
for c in C3 C5; do for k in 2 4 8 16 32 64; do
  r=$(python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-chunks $k 2>/dev/null | tail -1)
  echo "$c chunks $k $(echo "$r" | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print(e['value'], 'MP/s', e['ms_per_step'], 'ms')")"
done; done
