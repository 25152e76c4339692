"""Aggregate ncu warp-stall samples per CUDA source line (report captured with -lineinfo and
--import-source on): total samples, instructions executed and the top stall reasons per line.
    usage: python tools/ncu_lines.py REPORT.ncu-rep [top] [reason]
reason (e.g. long_sb, membar, wait): rank lines by that stall reason instead of all samples."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
key_reason = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


agg = collections.defaultdict(collections.Counter)
src = {}
hdr, fname = None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "":   # SASS rows repeat the line's samples
        continue
    d = dict(zip(hdr[4:], r[4:]))
    k = (fname, r[0])
    src[k] = r[1][:80]
    agg[k]["_all"] += num(d.get("Warp Stall Sampling (All Samples)", 0))
    agg[k]["_inst"] += num(d.get("Instructions Executed", 0))
    for name, v in d.items():
        if name.startswith("stall_") and "Not Issued" not in name:
            agg[k][name[6:]] += num(v)
tot = sum(c["_all"] for c in agg.values())
print(f"total samples {tot:.0f}")
rank = (lambda c: c[key_reason]) if key_reason else (lambda c: c["_all"])
for k, c in sorted(agg.items(), key=lambda kv: -rank(kv[1]))[:top]:
    rs = sorted(((v, n) for n, v in c.items() if not n.startswith("_") and v), reverse=True)[:3]
    print(f"{k[0]}:{k[1]:>5} {c['_all']:6.0f}  inst {c['_inst']:9.0f}  " + " ".join(f"{n}:{v:.0f}" for v, n in rs)
          + f"  | {src[k]}")
