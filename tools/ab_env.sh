# A/B of environment settings (policy knobs HR_<KEY>) on bench configs (gpurun, repo root):
#   bash tools/ab_env.sh "C5 C3" "" "HR_HIST_CPSM=1" ...   ("" = defaults)
cfgs=$1; shift
for c in $cfgs; do
  for envs in "$@"; do
    r=$(env $envs python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
    echo "$c [$envs] $(echo "$r" | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timing']; s=d['stages_ms_separate_kernels_info']; print(d['ms_per_step'], 'p50', t['median_ms'], 'hist', s['hist'], 'apply', s['apply'], 'solve', s['solve'])")"
  done
done
