# one ncu --set full capture of a kernel on a bench config (run with gpurun from the repo root):
#   bash tools/prof_one.sh <kernel regex> <config> <out name> [ENV=VAL ...]
mkdir -p gpurun_out
K=$1; C=$2; O=$3; shift 3
B="python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
env "$@" $B > /dev/null 2>&1 || { echo plain failed; exit 1; }
env "$@" ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/$O -f $B > gpurun_out/$O.log 2>&1
ls -la gpurun_out/$O.ncu-rep
