# A/B of an hr_enhance policy knob on the bench configs (run with gpurun from the repo root):
#   bash tools/ab_run.sh ENVVAR "v1 v2" "C3 C5" [pytest -k expr]
mkdir -p gpurun_out
VAR=${1:-HR_HIST_TMA}; VALS=${2:-"1 0"}; CFGS=${3:-"C3 C5"}; K=${4:-histogram}
python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "$K" > gpurun_out/ab_pytest.log 2>&1; tail -2 gpurun_out/ab_pytest.log
for c in $CFGS; do
  for t in $VALS; do env $VAR=$t python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_$t.json 2>gpurun_out/ab_${c}_$t.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_${c}_$t.json')); print('$c $VAR=$t', d['ms_per_step'], d['hbm_roofline_frac_e2e'], d['stages_ms'])"
  done
done
