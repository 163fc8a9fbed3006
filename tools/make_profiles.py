"""Copy one gpu_measure.sh result set from gpurun_out/ into profiles/ (tracked summaries).

    python tools/make_profiles.py <gpurun_out prefix> <profiles tag>     e.g. r02f r02

Bench lines -> profiles/<tag>_bench/Cx.json; ncu launch lists -> per-step summaries
(tools/ncu_steps.py) + the step's DRAM bytes into profiles/ncu_traffic.json (bench.py's roofline
"traffic"); full captures -> key-metric summaries (tools/ncu_summary.py); solver scans copied.
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src, tag = sys.argv[1], sys.argv[2]
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
PX = {"C1": 10000, "C2": 664000, "C3": 132710400, "C4": 33177600, "C5": 61440000}
os.makedirs(os.path.join(P, f"{tag}_bench"), exist_ok=True)
for c in PX:
    f = os.path.join(G, f"{src}_bench_{c}.json")
    if os.path.exists(f):
        shutil.copy(f, os.path.join(P, f"{tag}_bench", f"{c}.json"))
tj = os.path.join(P, "ncu_traffic.json")
traffic = json.load(open(tj)) if os.path.exists(tj) else {}
for c in PX:
    f = os.path.join(G, f"{src}_launches_{c}.csv")
    if not os.path.exists(f):
        continue
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_steps.py"), f, str(PX[c])],
                         capture_output=True, text=True).stdout
    name = f"{tag}_launches_{c}.txt"
    open(os.path.join(P, name), "w").write(out)
    last = json.loads(out.strip().splitlines()[-1])
    traffic[c] = {"step": last["step_dram_bytes"], "source": f"profiles/{name} (ncu launch list, last of 4 steps)"}
json.dump(traffic, open(tj, "w"), indent=1)
reps = {"k_hist_c3": "C3:k_hist", "k_apply_c3": "C3:k_apply", "k_solve_c3": "C3:k_solve",
        "k_hist_c5_full": "C5full:k_hist", "k_solve_cluster_c4": "C4:k_solve_cluster"}
args = []
for k, spec in reps.items():
    f = os.path.join(G, f"{src}_prof_{k}.ncu-rep")
    if os.path.exists(f):
        args.append(f"{f}:{spec}")
if args:
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), "--tag", tag, "--rep"] + args)
    # ncu_summary also records per-kernel traffic; keep only the per-step entries bench.py reads
    t = json.load(open(tj))
    for c in list(t):
        t[c] = {k: v for k, v in t[c].items() if k in ("step", "source")}
        if not t[c]:
            del t[c]
    json.dump(t, open(tj, "w"), indent=1)
for n in ("solve_scan", "cluster_scan"):
    f = os.path.join(G, f"{src}_{n}.txt")
    if os.path.exists(f):
        shutil.copy(f, os.path.join(P, f"{tag}_{n}.txt"))
print("profiles updated:", tag)
