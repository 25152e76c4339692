"""Summarise an ncu launch-list CSV (gpu__time_duration / dram bytes per launch) by kernel.
usage: python tools/launch_summary.py gpurun_out/launches_TAG.csv [steps_in_capture]"""
import collections
import csv
import sys

path = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hi], rows[hi + 1:]
iN, iM, iV, iID = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
k = collections.OrderedDict()
for r in data:
    k.setdefault((int(r[iID]), r[iN]), {})[r[iM]] = float(r[iV].replace(",", ""))
tot = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
allt = 0.0
for (_, n), m in k.items():
    nm = n.split("(")[0].replace("void ", "")[:58]
    t = m.get("gpu__time_duration.sum", 0.0)
    tot[nm][0] += 1
    tot[nm][1] += t
    tot[nm][2] += m.get("dram__bytes_read.sum", 0.0)
    tot[nm][3] += m.get("dram__bytes_write.sum", 0.0)
    allt += t
print(f"launches {len(k)} ({len(k) / steps:.0f} per step), serialized cold-cache ms per step {allt / 1e6 / steps:.3f}")
print(f"{'kernel':58s} {'n/step':>7s} {'ms/step':>8s} {'share':>6s} {'GB/s':>8s}")
for nm, (c, t, r, w) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"{nm:58s} {c / steps:7.1f} {t / 1e6 / steps:8.3f} {t / allt:6.3f} {(r + w) / t:8.1f}")
