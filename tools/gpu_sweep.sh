# execution-policy sweep (chunks x grids x solver), C3 and C5
for cfg in C3 C5; do
for ws in 0 1; do
for ch in 1 4 8; do
for hc in 2 1; do
  if [ "$ch" = "1" ] && [ "$hc" = "1" ]; then continue; fi
  r=$(HR_WARP_SOLVER=$ws HR_CHUNKS=$ch HR_HIST_CPSM=$hc HR_APPLY_CPSM=$hc python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['hbm_roofline_frac_e2e'])")
  echo "$cfg warp=$ws chunks=$ch cpsm=$hc -> $r"
done; done; done; done
