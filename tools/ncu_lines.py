"""Per-source-line warp-stall samples of one kernel from an ncu report (measurement tool).

ncu's source page is per SASS instruction; this maps each instruction to the CUDA source line
nvdisasm -g attributes it to (the library is built with -lineinfo) and sums the samples.

  python tools/ncu_lines.py <report.ncu-rep> <kernel substring> [lib.so] [top N]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_lines(lib, kname):
    """{offset: (file, line)} for the first function whose name contains kname."""
    tmp = tempfile.mkdtemp()
    if lib.endswith(".cubin"):
        import shutil

        shutil.copy(lib, tmp)
    else:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    out = {}
    for f in sorted(os.listdir(tmp)):
        if not f.endswith(".cubin"):
            continue
        dis = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, f)], capture_output=True, text=True).stdout
        infn, cur = False, None
        for ln in dis.splitlines():
            if ln.startswith("//----") and ".text." in ln:
                if infn:
                    return out
                infn = kname in ln
                continue
            if not infn:
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
            if m and cur:
                out[int(m.group(1), 16)] = cur
        if infn:
            return out
    return out


def main():
    rep, kname = sys.argv[1], sys.argv[2]
    lib = sys.argv[3] if len(sys.argv) > 3 else "paper_2510_21100_b200/libhistretinex.so"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    data = [r for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
    ci = {h: i for i, h in enumerate(hdr)}
    base = int(data[0][ci["Address"]], 16)
    lines = sass_lines(lib, kname)
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = collections.defaultdict(lambda: collections.Counter())
    total = 0
    for r in data:
        off = int(r[ci["Address"]], 16) - base
        key = lines.get(off, ("?", 0))
        s = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
        total += s
        c = agg[key]
        c["samples"] += s
        c["inst"] += int(r[ci["Instructions Executed"]] or 0)
        for h in stalls:
            v = r[ci[h]]
            if v and v != "0":
                c[h[6:]] += int(v)
    print(f"total samples {total}")
    for key, c in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
        det = ", ".join(f"{k} {v}" for k, v in c.most_common() if k not in ("samples", "inst"))[:110]
        print(f"{c['samples'] / max(total, 1) * 100:5.1f}% {key[0]}:{key[1]:<5} inst {c['inst']:>9}  {det}")


if __name__ == "__main__":
    main()
