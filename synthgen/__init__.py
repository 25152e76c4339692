"""Seeded synthetic input generators shared by the tests, the bench and smoke().

This module holds none of the method's arithmetic: it only draws random
numbers with the shapes and distributions of the paper's workloads (recipe in
DESIGN.md section 5).  Both the oracle and the CUDA path consume what it
produces; neither is imported here.

Recipe (reading R19):
  * frames: k/255 with k ~ U{0..255} (8-bit video), NCHW [T,3,H,W]      seed 2
  * latents / contexts: N(0,1), NHWC [T,h,w,256]                         seed 1
  * conv W, b ~ U(+-1/sqrt(fan_in)) (PyTorch default conv init)          seed 0
  * GroupNorm gamma ~ U(0.5, 1.5), beta ~ U(-0.5, 0.5)  (beta != 0 so the
    chain-start slice SiLU(beta) of reading R8 is observable)
Arrays are float32; callers cast to the device dtype and hand the oracle the
exact (cast) values.
"""
from __future__ import annotations

import numpy as np

SEED_WEIGHTS, SEED_INPUTS, SEED_FRAMES = 0, 1, 2


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def frames_u8(T: int, H: int, W: int, seed: int = SEED_FRAMES) -> np.ndarray:
    """Synthetic 8-bit RGB frames, NCHW [T,3,H,W] uint8."""
    return rng(seed).integers(0, 256, size=(T, 3, H, W), dtype=np.uint8)


def frames_u8_hwc(T: int, H: int, W: int, seed: int = SEED_FRAMES) -> np.ndarray:
    """The same 8-bit frames in the HWC layout of decoded video, [T,H,W,3] uint8."""
    return np.ascontiguousarray(frames_u8(T, H, W, seed).transpose(0, 2, 3, 1))


def frames(T: int, H: int, W: int, seed: int = SEED_FRAMES) -> np.ndarray:
    """Frames in [0,1] as k/255 (float32), NCHW [T,3,H,W]."""
    return (frames_u8(T, H, W, seed).astype(np.float64) / 255.0).astype(np.float32)


def normal(shape, seed: int = SEED_INPUTS, scale: float = 1.0) -> np.ndarray:
    return (rng(seed).standard_normal(size=shape) * scale).astype(np.float32)


def _conv(g, cout, k, cin):
    bound = 1.0 / np.sqrt(cin * k * k)
    w = g.uniform(-bound, bound, size=(cout, k, k, cin)).astype(np.float32)   # OHWI
    b = g.uniform(-bound, bound, size=(cout,)).astype(np.float32)
    return w, b


def _gn(g, c):
    return (g.uniform(0.5, 1.5, size=(c,)).astype(np.float32),
            g.uniform(-0.5, 0.5, size=(c,)).astype(np.float32))


def resblock_weights(cin: int, cout: int, seed: int = SEED_WEIGHTS, g=None) -> dict:
    """One ResBlock's parameters in the order of include/dvc.h's dvc_resblock."""
    g = rng(seed) if g is None else g
    d = {}
    d["gn1_w"], d["gn1_b"] = _gn(g, cin)
    d["conv1_w"], d["conv1_b"] = _conv(g, cout, 3, cin)
    d["gn2_w"], d["gn2_b"] = _gn(g, cout)
    d["conv2_w"], d["conv2_b"] = _conv(g, cout, 3, cout)
    if cin != cout:
        w, b = _conv(g, cout, 1, cin)
        d["sc_w"], d["sc_b"] = w.reshape(cout, cin), b
    else:
        d["sc_w"] = d["sc_b"] = None
    return d


RB_ORDER = ("gn1_w", "gn1_b", "conv1_w", "conv1_b", "gn2_w", "gn2_b",
            "conv2_w", "conv2_b", "sc_w", "sc_b")


def _linear(g, cout, cin, bias=True):
    bound = 1.0 / np.sqrt(cin)
    w = g.uniform(-bound, bound, size=(cout, cin)).astype(np.float32)
    b = g.uniform(-bound, bound, size=(cout,)).astype(np.float32) if bias else None
    return w, b


TF_ORDER = ("gn_w", "gn_b", "proj_in_w", "proj_in_b", "ln1_w", "ln1_b", "qkv_w", "out_w", "out_b",
            "ln2_w", "ln2_b", "ff1_w", "ff1_b", "ff2_w", "ff2_b", "proj_out_w", "proj_out_b")


def transformer_weights(C: int, seed: int = SEED_WEIGHTS, g=None, qkv_scale: float = 1.0) -> dict:
    """One Transformer2D block's parameters (reading R24; blob order TF_ORDER):
    Linear layers PyTorch-default U(+-1/sqrt(fan_in)); norms gamma ~ U(0.5,1.5),
    beta ~ U(-0.5,0.5).  qkv_scale > 1 sharpens the attention (test-only knob)."""
    g = rng(seed) if g is None else g
    d = {}
    d["gn_w"], d["gn_b"] = _gn(g, C)
    d["proj_in_w"], d["proj_in_b"] = _linear(g, C, C)
    d["ln1_w"], d["ln1_b"] = _gn(g, C)
    d["qkv_w"], _ = _linear(g, 3 * C, C, bias=False)
    d["qkv_w"] = (d["qkv_w"] * qkv_scale).astype(np.float32)
    d["out_w"], d["out_b"] = _linear(g, C, C)
    d["ln2_w"], d["ln2_b"] = _gn(g, C)
    d["ff1_w"], d["ff1_b"] = _linear(g, 8 * C, C)
    d["ff2_w"], d["ff2_b"] = _linear(g, C, 4 * C)
    d["proj_out_w"], d["proj_out_b"] = _linear(g, C, C)
    return d


def expansion_weights(c_lat: int = 256, c_in: int = 192, seed: int = SEED_WEIGHTS):
    """Encoder-side Latent Channel Expansion 1x1 conv (reading R13): W [c_lat, c_in], b."""
    w, b = _conv(rng(seed), c_lat, 1, c_in)
    return w.reshape(c_lat, c_in), b


def unet_weights(width=(240, 480, 960, 960), c_lat: int = 256, c_ctx: int = 256,
                 seed: int = SEED_WEIGHTS, attention: bool = False, qkv_scale: float = 1.0):
    """All skeleton tensors as [(name, float32 array)] in the blob order that
    include/dvc.h documents for dvc_unet_create:
      conv_in{w,b}; the 22 ResBlocks in U-Net order, each
      {gn1_w,gn1_b,conv1_w,conv1_b,gn2_w,gn2_b,conv2_w,conv2_b[,sc_w,sc_b]}, with the
      stride-2 conv{w,b} after down_l.r1 (l<3) and the post-upsample conv{w,b}
      after up_u.r2 (u<3); then gn_out{w,b}; conv_out{w,b}.
    attention=True (full U-Net, f1): a Transformer2D block's tensors (TF_ORDER) follow
      every ResBlock of down levels 0-2, mid.r0 and every ResBlock of up levels 2-0."""
    g = rng(seed)
    out = []

    def conv(name, cout, cin, k=3):
        w, b = _conv(g, cout, k, cin)
        out.append((name + ".w", w))
        out.append((name + ".b", b))

    def block(name, cin, cout):
        d = resblock_weights(cin, cout, g=g)
        for k in RB_ORDER:
            if d[k] is not None:
                out.append((f"{name}.{k}", d[k]))

    def tf(name, C):
        if attention:
            d = transformer_weights(C, g=g, qkv_scale=qkv_scale)
            for k in TF_ORDER:
                out.append((f"{name}.tf.{k}", d[k]))

    conv("conv_in", width[0], c_lat + c_ctx)
    skip_ch = [width[0]]
    cur = width[0]
    for l in range(4):
        for r in range(2):
            block(f"down{l}.r{r}", cur, width[l])
            cur = width[l]
            if l < 3:
                tf(f"down{l}.r{r}", cur)
            skip_ch.append(cur)
        if l < 3:
            conv(f"down{l}.ds", cur, cur)
            skip_ch.append(cur)
    for r in range(2):
        block(f"mid.r{r}", cur, cur)
        if r == 0:
            tf("mid.r0", cur)
    for u in range(4):
        lvl = 3 - u
        for r in range(3):
            block(f"up{u}.r{r}", cur + skip_ch.pop(), width[lvl])
            cur = width[lvl]
            if u > 0:
                tf(f"up{u}.r{r}", cur)
        if u < 3:
            conv(f"up{u}.us", cur, cur)
    gw, gb = _gn(g, cur)
    out.append(("gn_out.w", gw))
    out.append(("gn_out.b", gb))
    conv("conv_out", c_lat, cur)
    return out


def vae_weights(width=(64, 128, 256, 256), c_lat: int = 256, out_ch: int = 3, mid_attn: bool = True,
                seed: int = SEED_WEIGHTS, attn_scale: float = 1.0):
    """Pruned VAE decoder tensors (f2, reading R29) in the blob order of include/dvc.h's
    dvc_vae_create: conv_in{w,b}; mid.r0; [mid attention {gn_w, gn_b, q_w, q_b, k_w, k_b, v_w, v_b,
    out_w, out_b}]; mid.r1; for each up level i (widths reversed) 3 ResBlocks then (i < 3) the
    post-upsample conv{w,b}; gn_out{w,b}; conv_out{w,b}.  ResBlocks as in resblock_weights."""
    g = rng(seed)
    out = []

    def conv(name, cout, cin, k=3):
        w, b = _conv(g, cout, k, cin)
        out.append((name + ".w", w))
        out.append((name + ".b", b))

    def block(name, cin, cout):
        d = resblock_weights(cin, cout, g=g)
        for k in RB_ORDER:
            if d[k] is not None:
                out.append((f"{name}.{k}", d[k]))

    top = width[-1]
    conv("conv_in", top, c_lat)
    block("mid.r0", top, top)
    if mid_attn:
        gw, gb = _gn(g, top)
        out += [("mid.attn.gn_w", gw), ("mid.attn.gn_b", gb)]
        for nm in ("q", "k", "v", "out"):
            w, b = _linear(g, top, top)
            if nm in ("q", "k"):
                w = (w * attn_scale).astype(np.float32)
            out += [(f"mid.attn.{nm}_w", w), (f"mid.attn.{nm}_b", b)]
    block("mid.r1", top, top)
    cur = top
    for i, c in enumerate(reversed(width)):
        for r in range(3):
            block(f"up{i}.r{r}", cur, c)
            cur = c
        if i < 3:
            conv(f"up{i}.us", c, c)
    gw, gb = _gn(g, cur)
    out += [("gn_out.w", gw), ("gn_out.b", gb)]
    conv("conv_out", out_ch, cur)
    return out

