"""f1 measurements (one GPU), one JSON line each:

    python tools/bench_f1.py [--quick]

  ATTN  the tcgen05 attention kernel alone at the 720p U-Net shapes (T=32 frames: level 0
        N=14400 C=240, level 1 N=3600 C=480, level 2 N=920 C=960, head_dim 48): ms, algorithmic
        TFLOP/s (4*N^2*C per frame) and the fraction of the measured bf16 peaks
  F1    full pruned U-Net (22 ResBlocks + 16 Transformer2D blocks, R24-R26) decode at 720p,
        T=32, bf16: frames/s, and the per-kernel-family split of one profiled step
The headline metric (bench.py) stays the ResBlock-skeleton decode the north star names.
"""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2601_20564_b200 as dvc  # noqa: E402
import synthgen  # noqa: E402

WIDTH = (240, 480, 960, 960)


def timed(fn, steps, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return p["bf16_tflops"], p["bf16_tflops_sustained"]
    except Exception:
        return 1663.0, 1400.0


def attn(steps):
    burst, sus = peaks()
    rows = []
    for lvl, (N, C) in enumerate(((14400, 240), (3600, 480), (920, 960))):
        T = 32
        qkv = torch.from_numpy(synthgen.normal((T, N, 3 * C), 11)).to(torch.bfloat16).cuda()
        out = torch.empty((T, N, C), dtype=torch.bfloat16, device="cuda")
        ws = None   # the library sizes and allocates its packed-operand workspace
        dvc.profile_begin()
        ms = timed(lambda: dvc.dvc_attention_forward(qkv, 48, out=out, workspace=ws), steps)
        dvc.profile_end()
        recs = dvc.profile_records()
        k_ms = [r[1] for r in recs if r[0].startswith("attn_tc")]
        kms = sum(k_ms) / max(1, len(k_ms))
        fl = 4.0 * T * N * N * C
        rows.append({"level": lvl, "T": T, "N": N, "C": C, "heads": C // 48, "call_ms": ms, "kernel_ms": kms,
                     "tflops": fl / (kms / 1e3) / 1e12, "frac_burst": fl / (kms / 1e3) / 1e12 / burst,
                     "frac_sustained": fl / (kms / 1e3) / 1e12 / sus})
    return {"config": "ATTN tcgen05 attention, 720p U-Net shapes, T=32, bf16, head_dim 48", "rows": rows}


def full_unet(steps, T=32, h=90, w=160):
    named = synthgen.unet_weights(WIDTH, 256, 256, attention=True)
    cfg = dvc.unet_config(WIDTH, 256, 256, 24, 8, 1e-5, torch.bfloat16, h, w, T, head_dim=48)
    net = dvc.UNet(cfg, dvc.pack_weights(named, torch.bfloat16))
    lat = torch.from_numpy(synthgen.normal((T, h, w, 256), 1)).to(torch.bfloat16).cuda()
    ctx = torch.from_numpy(synthgen.normal((T, h, w, 256), 5)).to(torch.bfloat16).cuda()
    out = torch.empty_like(lat)
    ws = torch.empty(net.workspace_size(T), dtype=torch.uint8, device="cuda")
    run = lambda: dvc.dvc_unet_decode_gop(net, lat, ctx, out=out, workspace=ws)  # noqa: E731
    ms = timed(run, steps)
    dvc.profile_begin()
    run()
    conv_ms, conv_fl, nconv = dvc.profile_end()
    fam = collections.defaultdict(lambda: [0.0, 0.0, 0])
    for lab, kms, fl in dvc.profile_records():
        key = lab.split(" ")[0]
        if key in ("ws", "tc", "fz1", "fz2", "fz_out", "simt"):
            key = "conv_" + ("1x1" if " K=" in lab and "segs=1" in lab and _is1x1(lab) else "3x3")
        fam[key][0] += kms
        fam[key][1] += fl
        fam[key][2] += 1
    burst, sus = peaks()
    split = {k: {"ms": v[0], "launches": v[2], "tflops": (v[1] / (v[0] / 1e3) / 1e12) if v[1] else None}
             for k, v in sorted(fam.items(), key=lambda kv: -kv[1][0])}
    return {"config": f"F1 full U-Net decode 720p T={T} bf16 (22 ResBlocks + 16 Transformer2D, head_dim 48)",
            "ms_per_step": ms, "frames_per_s": T / (ms / 1e3), "profiled_split": split,
            "conv_tflops": conv_fl / (conv_ms / 1e3) / 1e12, "peak_sustained": sus}


def _is1x1(lab):
    # conv labels: "<engine> T=.. HxW K=.. N=.. segs=..": the transformer linears have K = C_in (taps 1)
    try:
        k = int(lab.split("K=")[1].split(" ")[0])
    except Exception:
        return False
    return k in (240, 480, 960, 1920, 3840)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    steps = 3 if args.quick else 10
    print(json.dumps(attn(steps)), flush=True)
    print(json.dumps(full_unet(max(3, steps // 2))), flush=True)


if __name__ == "__main__":
    main()
