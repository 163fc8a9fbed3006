bash tools/ab_env.sh "C5" "X=0" "HR_GROUPS=3 HR_GROUP_SPLITS=60,90" "HR_GROUPS=3 HR_GROUP_SPLITS=75,94" "HR_GROUPS=3 HR_GROUP_SPLITS=50,85" "HR_GROUPS=3 HR_GROUP_SPLITS=85,96" > /dev/null 2>&1
for f in gpurun_out/abe_C5_[12345].json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d['ms_per_step'], d['hbm_roofline_frac_e2e'])"; done
bash tools/ab_env.sh "C3" "X=0" "HR_GROUPS=3 HR_GROUP_SPLITS=25,60" "HR_GROUPS=3 HR_GROUP_SPLITS=20,50" "HR_GROUPS=3 HR_GROUP_SPLITS=30,75" > /dev/null 2>&1
for f in gpurun_out/abe_C3_[1234].json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d['ms_per_step'], d['hbm_roofline_frac_e2e'])"; done
