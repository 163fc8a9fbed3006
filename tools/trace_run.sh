# step timelines under several settings (run with gpurun from the repo root):
#   CFGS="C3 C5" bash tools/trace_run.sh "ENV=V ..." "ENV=V ..."
export HR_LIB=tools/libhistretinex_steptrace.so
for c in ${CFGS:-C3 C5}; do
  for setting in "$@"; do python tools/step_trace.py $c $setting; done
done
