# A/B over arbitrary environment settings on bench configs (run with gpurun from the repo root):
#   bash tools/ab_env.sh "C3 C5" "A=1 B=2" "A=0" ...      (each quoted group is one setting)
mkdir -p gpurun_out
CFGS=$1; shift
for c in $CFGS; do
  i=0
  for setting in "$@"; do
    i=$((i+1))
    env $setting python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/abe_${c}_$i.json 2>gpurun_out/abe_${c}_$i.err
    python -c "
import json; d=json.load(open('gpurun_out/abe_${c}_$i.json')); s=d['stages_ms']; print('$c [$setting]', d['ms_per_step'], d['hbm_roofline_frac_e2e'], 'hist', s['hist'], 'solve', s['solve'], 'apply', s['apply'])" || tail -3 gpurun_out/abe_${c}_$i.err
  done
done
