"""Write the committed profile summaries from a gpurun_out capture.
usage: python tools/make_profiles.py TAG [ROUND]
  gpurun_out/launches_TAG.csv   (ncu --metrics gpu__time_duration.sum,dram__bytes_* launch list, 2 steps)
  gpurun_out/prof_convws_TAG.ncu-rep (ncu --set full, conv_ws launches)
  gpurun_out/bench_TAG.json     (bench line)"""
import collections
import csv
import json
import os
import subprocess
import sys

tag = sys.argv[1]
rnd = sys.argv[2] if len(sys.argv) > 2 else "r1"
G = "gpurun_out"
os.makedirs("profiles", exist_ok=True)

# ---- launch list
rows = list(csv.reader(open(f"{G}/launches_{tag}.csv")))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hi], rows[hi + 1:]
iN, iM, iV, iID = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
iG = hdr.index("Grid Size")
k = collections.OrderedDict()
for r in data:
    d = k.setdefault(int(r[iID]), {"name": r[iN].split("(")[0].replace("void ", ""), "grid": r[iG]})
    d[r[iM]] = float(r[iV].replace(",", ""))
items = list(k.values())
# one encode launch per bench step (warm-up, timed and instrumented passes are all in the capture)
steps = max(1, sum(1 for d in items if d["name"].startswith("encode_kernel")))
second = items[-(len(items) // steps):]
tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in items:
    t = d["gpu__time_duration.sum"]
    b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    tot[d["name"]][0] += 1
    tot[d["name"]][1] += t
    tot[d["name"]][2] += b
allt = sum(v[1] for v in tot.values())
conv_bytes = sum(v[2] for n, v in tot.items() if "conv_" in n) / steps
conv_ns = sum(v[1] for n, v in tot.items() if "conv_" in n) / steps
with open(f"profiles/{rnd}_launches.txt", "w") as f:
    f.write(f"# ncu launch list ({tag}): ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
            f"--clock-control none -c 500 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline\n"
            f"# {steps} steps captured (warm-up, timed and instrumented passes); times are serialized, "
            f"cold-cache (ncu flushes caches): "
            f"compare SHARES with bench.py, not absolutes\n")
    f.write(f"# launches per step {len(items) / steps:.0f}; serialized ms per step {allt / 1e6 / steps:.3f}\n")
    f.write(f"{'kernel':60s} {'n/step':>7s} {'ms/step':>8s} {'share':>6s} {'DRAM GB/s':>10s}\n")
    for n, (c, t, b) in sorted(tot.items(), key=lambda x: -x[1][1]):
        f.write(f"{n[:60]:60s} {c / steps:7.1f} {t / 1e6 / steps:8.3f} {t / allt:6.3f} {b / t:10.1f}\n")
    f.write("\n# per launch, timed step\n")
    for d in second:
        t = d["gpu__time_duration.sum"]
        b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        f.write(f"{d['name'][:48]:48s} {d['grid']:>14s} {t / 1e3:9.1f} us {b / 1e6:9.1f} MB\n")
json.dump({"bytes_per_step": conv_bytes, "conv_ns_per_step_ncu": conv_ns,
           "source": f"profiles/{rnd}_launches.txt (sum of dram__bytes_read+write over all conv launches of one step)"},
          open("profiles/traffic.json", "w"), indent=1)

# ---- full captures of the conv kernels
for eng, what in (("ws", "launch 0 = conv_in, launch 1 = the first persistent-TMA ResBlock conv"),
                  ("fz", "launch 0 = down0.r0 conv1 (fused GN/SiLU/shift), launch 1 = its conv2 (+ identity skip)")):
  rep = f"{G}/prof_conv{eng}_{tag}.ncu-rep"
  if os.path.exists(rep):
      raw = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
      r = list(csv.reader(raw.splitlines()))
      h = r[0]
      keep = ("Duration", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
              "Compute (SM) Throughput", "Registers Per Thread", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block",
              "Achieved Occupancy", "L2 Hit Rate", "Issue Slots Busy")
      with open(f"profiles/{rnd}_conv_{eng}_full.txt", "w") as f:
          f.write(f"# ncu --set full --clock-control none --import-source on -k regex:conv_{eng} -s 0 -c 2 ({what}, "
                  f"720p T=32 bf16)\n")
          for row in r[1:]:
              d = dict(zip(h, row))
              if d.get("Metric Name") in keep:
                  f.write(f"launch {d['ID']}  {d['Metric Name']:35s} {d['Metric Value']:>14s} {d['Metric Unit']}\n")
          raw2 = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
          r2 = list(csv.reader(raw2.splitlines()))
          for row in r2[2:]:
              d = dict(zip(r2[0], row))
              for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "lts__t_bytes.sum"):
                  if m in d:
                      f.write(f"raw {m:80s} {d[m]} {r2[1][r2[0].index(m)]}\n")
for extra in ("breakdown", "fzprof"):
    src = f"{G}/{extra}_{tag}.txt"
    if os.path.exists(src):
        lines = open(src).read().splitlines()
        if extra == "fzprof":
            lines = lines[-20:]
        open(f"profiles/{rnd}_{extra}.txt", "w").write("\n".join(lines) + "\n")
bj = f"{G}/bench_{tag}.json"
if os.path.exists(bj):
    line = [l for l in open(bj) if l.startswith("{")][-1]
    open(f"profiles/{rnd}_bench.json", "w").write(line)
print("ok", conv_bytes / 1e9, "GB conv dram per step")
