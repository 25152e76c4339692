"""Helpers shared by the -m gpu parity tests (no method arithmetic here)."""
import numpy as np
import torch

MODE = {torch.bfloat16: "bf16", torch.float16: "fp16", torch.float32: None}
TOL = {torch.bfloat16: 1e-2, torch.float16: 1e-2, torch.float32: 1e-5}   # north_star tolerances (R16)


def dev(a, dtype):
    """numpy float32 -> device tensor of dtype, plus the exact fp64 values the device holds."""
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dtype)
    return t.cuda(), t.double().numpy()


def host64(t):
    return t.detach().double().cpu().numpy()


def rb_device(w: dict, dtype):
    """synthgen ResBlock weights -> (device tensors, exact fp64 copies for the oracle)."""
    d, h = {}, {}
    for k, v in w.items():
        if v is None:
            d[k] = h[k] = None
        else:
            d[k], h[k] = dev(v, dtype)
    return d, h


def rel_l2(a, ref):
    a, ref = np.asarray(a, np.float64), np.asarray(ref, np.float64)
    return float(np.linalg.norm((a - ref).ravel()) / max(np.linalg.norm(ref.ravel()), 1e-300))
