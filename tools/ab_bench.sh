# A/B of library builds on bench configs (run with gpurun from the repo root):
#   bash tools/ab_bench.sh "C5 C3" lib1.so lib2.so ...   (a lib named "-" = the product build)
cfgs=$1; shift
for c in $cfgs; do
  for lib in "$@"; do
    if [ "$lib" = "-" ]; then L=""; else L="$lib"; fi
    r=$(HR_LIB=$L python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
    echo "$c $lib $(echo "$r" | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; s=d['stages_ms_separate_kernels_info']; print(d['ms_per_step'], 'p50', t['median_ms'], 'hist', s['hist'], 'apply', s['apply'], 'solve', s['solve'])")"
  done
done
