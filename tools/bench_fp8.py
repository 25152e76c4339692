"""f4 fp8 measurement (one GPU): the same 3x3 convolutions in bf16 and in fp8 (E4M3 operands,
kind::f8f6f4), at the 720p U-Net shapes with 32 frames, one JSON line.

    python tools/bench_fp8.py

TFLOP/s are algorithmic (2*M*N*K) over the CUDA-event time of the kernel; the fp8 peak is the
measured bf16 dense peak x 2 (the nominal 4.5 / 2.25 PF ratio, B200_PROFILING.md).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_20564_b200 as dvc  # noqa: E402
import synthgen  # noqa: E402


def kernel_ms(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dvc.profile_begin()
    for _ in range(reps):
        fn()
    dvc.profile_end()
    r = [x for x in dvc.profile_records() if x[0].startswith("ws") or x[0].startswith("tc")]
    return sum(x[1] for x in r) / len(r), r[0][2]


def main():
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops_sustained"]
    except Exception:
        pk = 1364.1
    rows = []
    for (lvl, H, W, C) in ((1, 45, 80, 480), (2, 23, 40, 960), (3, 12, 20, 960)):
        T = 32
        x = torch.from_numpy(synthgen.normal((T, H, W, C), 1)).to(torch.bfloat16).cuda()
        w = torch.from_numpy(synthgen.normal((C, 3, 3, C), 2, scale=1 / np.sqrt(9 * C))).to(torch.bfloat16).cuda()
        b = torch.zeros(C, dtype=torch.bfloat16, device="cuda")
        sx, sw = float(x.abs().max()) / 448, float(w.abs().max()) / 448
        x8, w8 = dvc.dvc_quantize_e4m3(x, sx), dvc.dvc_quantize_e4m3(w, sw)
        y = torch.empty((T, H, W, C), dtype=torch.bfloat16, device="cuda")
        ms8, fl = kernel_ms(lambda: dvc.dvc_conv_fp8(x8, sx, w8, sw, b, out=y))
        ms16, fl16 = kernel_ms(lambda: dvc.dvc_conv(x, w, b, out=y))
        rows.append({"level": lvl, "T": T, "HxW": f"{H}x{W}", "C": C, "fp8_ms": ms8, "fp8_tflops": fl / ms8 / 1e9,
                     "fp8_frac_of_2x_bf16_sustained": fl / ms8 / 1e9 / (2 * pk),
                     "bf16_ms": ms16, "bf16_tflops": fl16 / ms16 / 1e9, "bf16_frac_sustained": fl16 / ms16 / 1e9 / pk,
                     "speedup": ms16 / ms8})
    print(json.dumps({"config": "F4 fp8 vs bf16 3x3 conv, 720p U-Net level shapes, T=32 (E4M3 in, bf16 out)",
                      "rows": rows, "fp8_peak_used": 2 * pk}), flush=True)


if __name__ == "__main__":
    main()
