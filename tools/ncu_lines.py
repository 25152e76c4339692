"""Aggregate ncu warp-stall samples per CUDA source line (report captured with -lineinfo and
--import-source on).  usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_INDEX [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kid = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
lo, hi = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else (0, 1 << 30)   # line filter (main file)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-id", f":::{kid}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = collections.defaultdict(lambda: collections.Counter())
src = {}
fname, hdr = None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name", ""):
        continue
    nm = len(hdr) - 4   # metric columns are the trailing ones (source text may contain stray quotes)
    d = {k: v for k, v in zip(hdr[4:], r[-nm:]) if v not in ("-", "")}
    try:
        line = int(r[0])
    except ValueError:
        continue
    key = (fname, line)
    src[key] = r[1][:70]
    s = float(d.get("Warp Stall Sampling (All Samples)") or 0)
    agg[key]["_all"] += s
    agg[key]["_inst"] += float(d.get("Instructions Executed") or 0)
    for k, v in d.items():
        if k.startswith("stall_") and "Not" not in k and v:
            agg[key][k] += float(v)
tot = sum(c["_all"] for c in agg.values())
print(f"total samples {tot:.0f}")
sel = [kv for kv in agg.items() if len(sys.argv) <= 5 or (kv[0][0].endswith(".cu") and lo <= kv[0][1] <= hi)]
if len(sys.argv) > 5:
    print(f"lines {lo}-{hi}: {sum(c['_all'] for _, c in sel):.0f} samples")
for key, c in sorted(sel, key=lambda x: -x[1]["_all"])[:top]:
    reasons = sorted(((v, k[6:]) for k, v in c.items() if k.startswith("stall_")), reverse=True)[:3]
    rs = " ".join(f"{k}:{v:.0f}" for v, k in reasons)
    print(f"{c['_all']:7.0f} {100 * c['_all'] / tot:5.1f}% {key[0][:16]}:{key[1]:<4d} {src[key]:70s} {rs}")
