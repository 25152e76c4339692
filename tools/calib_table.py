"""Merge the ncu calibration captures (tools/gpu_calib.sh) into one table: for the cuBLAS 8192^3 bf16
GEMM and every conv launch of one 720p bench step, the algorithmic FLOPs (the library's own records),
ncu duration and SM clock, and three utilisation figures:
  alg/clk  = FLOPs / (duration x SM clock x 148 SMs x 8192 dense bf16 FLOP/clk/SM)   (clock-normalised)
  tensor%  = TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime (pct of peak sustained elapsed)
  tmem%    = sm__mem_tensor_cycles_active (pct of peak sustained elapsed)
usage: python tools/calib_table.py gpurun_out/calib  > profiles/r2_tensor_pipe_calibration.txt"""
import csv
import io
import json
import sys

PEAK_PER_CLK = 148 * 8192          # dense bf16 FLOP per clock per GPU (2.25 PF at 1.855 GHz x 148 SMs)


def load(path):
    lines = [ln for ln in open(path).read().splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr, out = rows[0], {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        k = int(d["ID"])
        e = out.setdefault(k, {"name": d["Kernel Name"]})
        e[d["Metric Name"]] = d["Metric Value"]
    return [out[k] for k in sorted(out)]


def f(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


def row(label, flops, m):
    dur = f(m["gpu__time_duration.sum"]) * 1e-9
    clk = f(m["sm__cycles_elapsed.avg.per_second"])
    alg = flops / (dur * clk * PEAK_PER_CLK)
    tp = f(m.get("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"))
    tm = f(m.get("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"))
    return (f"{label:46s} {flops / 1e9:8.1f} {dur * 1e6:8.1f} {clk / 1e9:5.2f} {flops / dur / 1e12:7.0f} "
            f"{100 * alg:6.1f} {tp:6.1f} {tm:6.1f}"), alg, tp, dur


pre = sys.argv[1]
gemm = [m for m in load(pre + "_gemm.csv") if "gemm" in m["name"].lower() or "nvjet" in m["name"].lower()]
conv = load(pre + "_conv.csv")
recs = json.load(open(pre + "_flops.json"))
print(f"{'launch':46s} {'GFLOP':>8s} {'us':>8s} {'GHz':>5s} {'TF/s':>7s} {'alg/clk':>6s} {'tensor%':>6s} {'tmem%':>6s}")
for m in gemm:
    print(row("cuBLAS bf16 8192^3 (" + m["name"][:20] + ")", 2 * 8192 ** 3, m)[0])
assert len(recs) == len(conv), (len(recs), len(conv))
tot_f = tot_t = 0.0
wa = wt = 0.0
for (lab, ms, fl), m in zip(recs, conv):
    line, alg, tp, dur = row(lab[:46], fl, m)
    print(line)
    tot_f += fl
    tot_t += dur
    wa += alg * dur
    wt += tp * dur
print(f"{'all conv launches (time-weighted)':46s} {tot_f / 1e9:8.1f} {tot_t * 1e6:8.1f} {'':5s} "
      f"{tot_f / tot_t / 1e12:7.0f} {100 * wa / tot_t:6.1f} {wt / tot_t:6.1f}")
