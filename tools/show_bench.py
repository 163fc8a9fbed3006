"""One line per bench JSON under gpurun_out/ (measurement helper)."""
import glob
import json
import sys

for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        print(f, "ERR")
        continue
    st = d.get("stages_ms_separate_kernels_info") or d.get("stages_ms") or d.get("stages_ms_unfused_info") or {}
    print(f"{f:38s} {d['value']:>10.1f} MP/s {d['ms_per_step']:.4f} ms  e2e_frac {d.get('hbm_roofline_frac_e2e')}"
          f"  {d['roofline']['kernel']} {d['roofline']['frac']}  "
          f"hist {st.get('hist')} solve {st.get('solve')} apply {st.get('apply')}  launches {d.get('gpu_launches')}  "
          f"p10/50/90 {(d.get('timing') or {}).get('p10_ms')}/{(d.get('timing') or {}).get('median_ms')}/"
          f"{(d.get('timing') or {}).get('p90_ms')}")
