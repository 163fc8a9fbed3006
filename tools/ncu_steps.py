"""Per-step summary of an ncu launch list (tools/gpu_measure.sh: --metrics gpu__time_duration,
dram__bytes_read/write over K hr_enhance steps): each step's kernels with their serialised,
cold-cache device time and DRAM bytes, and the step totals; the last step is the one reported.

    python tools/ncu_steps.py gpurun_out/r02c_launches_C3.csv [pixels]
"""
import csv
import json
import re
import sys
from collections import OrderedDict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "ID")
    ci = {h: i for i, h in enumerate(hdr)}
    out = OrderedDict()
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) != len(hdr):
            continue
        k = out.setdefault(int(r[ci["ID"]]), {"name": r[ci["Kernel Name"]], "grid": r[ci["Grid Size"]]})
        v = float(r[ci["Metric Value"]].replace(",", ""))
        k[r[ci["Metric Name"]]] = v
    return list(out.values())


def short(name):
    m = re.search(r"(k_[a-z0-9_]+)(<[^>]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:30]


def steps(ls):
    """Split at each k_zero launch that follows a non-k_zero launch (the start of a step)."""
    st, cur = [], []
    for i, k in enumerate(ls):
        z = short(k["name"]).startswith("k_zero")
        if z and cur and not short(ls[i - 1]["name"]).startswith("k_zero"):
            st.append(cur)
            cur = []
        cur.append(k)
    if cur:
        st.append(cur)
    return st


def main():
    path = sys.argv[1]
    px = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    ss = steps(launches(path))
    last = ss[-1]
    tot_t = sum(k.get("gpu__time_duration.sum", 0) for k in last)
    tot_b = sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in last)
    print(f"{path}: {len(ss)} steps; last step: {len(last)} launches, serialised device time {tot_t / 1e3:.1f} us, "
          f"DRAM {tot_b / 1e6:.1f} MB" + (f" ({tot_b / px:.2f} B/px vs 9 algorithmic)" if px else ""))
    for k in last:
        t = k.get("gpu__time_duration.sum", 0)
        b = k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
        print(f"  {short(k['name']):28s} grid {k['grid']:>14s} {t / 1e3:8.1f} us  {b / 1e6:9.2f} MB  "
              f"{(b / t if t else 0):7.1f} GB/s  share {t / tot_t * 100:5.1f}%")
    print(json.dumps({"step_dram_bytes": tot_b, "step_serialised_us": round(tot_t / 1e3, 2)}))


if __name__ == "__main__":
    main()
