"""fp64 oracle for the DiffVC-RT decode hot path (TEST INFRASTRUCTURE ONLY).

Plain, slow, obviously correct.  Heavy loops (conv, group norm, unshuffle,
rounding) live in ``dvc_oracle.c`` as direct loops; this module composes them
in exactly the order the paper / readings define.  Citations:
``P:<line>`` -> /root/reference/PAPER.md, ``S:<line>`` -> /root/reference/SPEC.md,
``R<n>`` -> readings in DESIGN.md section 3.

Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may use this module.  It never imports the product.

Parity status: every function below is pinned by a
``-m "not gpu"`` test in tests/test_oracle_pins.py (the a-rows) or
tests/test_oracle_attention.py (f1 Transformer2D / attention / GELU / LayerNorm,
f2 VAE decoder, f4 E4M3 rounding) except agreement with the paper's trained
model, which is unpinnable (no weights are published): the readings R2-R4, R8,
R11, R13, R24-R25, R29's 256-channel interface and R30 are "parity unpinned"
against the paper's numbers and pinned only structurally (the topologies are
pinned by Table 8's parameter counts).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dvc_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_LIB = None

_D = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile the C oracle (plain gcc, fp64, OpenMP).  Returns the .so path."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-std=c11",
               "-o", _SO + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


def lib():
    global _LIB
    if _LIB is None:
        _LIB = ctypes.CDLL(build())
        i, d, sz = ctypes.c_int, ctypes.c_double, ctypes.c_size_t
        _LIB.orc_unshuffle.argtypes = [_D, i, i, i, i, i, _D]
        _LIB.orc_shuffle.argtypes = [_D, i, i, i, i, i, _D]
        _LIB.orc_conv2d.argtypes = [_D, i, i, i, i, _D, _D, i, i, i, i, _D]
        _LIB.orc_groupnorm.argtypes = [_D, i, i, i, i, _D, _D, d, _D]
        _LIB.orc_silu.argtypes = [_D, sz, _D]
        _LIB.orc_nearest_to.argtypes = [_D, i, i, i, i, i, i, _D]
        _LIB.orc_round.argtypes = [_D, sz, i]
        _LIB.orc_round1.argtypes = [d, i]
        _LIB.orc_round1.restype = d
        _LIB.orc_num_threads.restype = i
    return _LIB


def _p(a):
    return a.ctypes.data_as(_D)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def num_threads() -> int:
    return lib().orc_num_threads()


# --------------------------------------------------------------------------
# precision emulation (R15)
# --------------------------------------------------------------------------
_MODES = {None: 0, "f32": 0, "fp16": 1, "bf16": 2}


def rnd(x, mode):
    """Round-to-nearest-even, directly from fp64, to binary16 ('fp16') or
    bfloat16 ('bf16'); identity for None / 'f32'.  Returns a new array."""
    x = _f64(x).copy()
    m = _MODES[mode]
    if m:
        lib().orc_round(_p(x), x.size, m)
    return x


def rnd1(v: float, mode) -> float:
    return lib().orc_round1(float(v), _MODES[mode])


# --------------------------------------------------------------------------
# a1. PixelUnshuffle (R12) and its inverse
# --------------------------------------------------------------------------
def unshuffle(F, s: int = 8):
    """F [T,C,H,W] -> L [T,H/s,W/s,C*s*s] with L[t,y,x,c*s*s+i*s+j] = F[t,c,s*y+i,s*x+j]."""
    F = _f64(F)
    T, C, H, W = F.shape
    if H % s or W % s:
        raise ValueError("divisibility error: H and W must be multiples of s (S:56)")
    L = np.empty((T, H // s, W // s, C * s * s))
    assert lib().orc_unshuffle(_p(F), T, C, H, W, s, _p(L)) == 0
    return L


def shuffle(L, C: int, s: int = 8):
    """Inverse of unshuffle: L [T,h,w,C*s*s] -> F [T,C,h*s,w*s]."""
    L = _f64(L)
    T, h, w, CL = L.shape
    if CL != C * s * s:
        raise ValueError("divisibility error: channels must be C*s*s")
    F = np.empty((T, C, h * s, w * s))
    assert lib().orc_shuffle(_p(L), T, C, h, w, s, _p(F)) == 0
    return F


# --------------------------------------------------------------------------
# R14: 8-bit HWC frames -> frame values u / 255 in the latent precision
# --------------------------------------------------------------------------
def _round_fraction(q, mode) -> float:
    """Round the exact rational q (fractions.Fraction, 0 <= q <= 1) to the nearest value of the
    format, ties to even: 'fp16' (11-bit significand), 'bf16' (8-bit) or 'f32' (24-bit)."""
    from fractions import Fraction
    import math
    bits = {"fp16": 11, "bf16": 8, "f32": 24}[mode]
    if q == 0:
        return 0.0
    e = math.floor(math.log2(q))
    if Fraction(2) ** e > q:          # guard the float log2 near powers of two
        e -= 1
    if Fraction(2) ** (e + 1) <= q:
        e += 1
    e = max(e, {"fp16": -14, "bf16": -126, "f32": -126}[mode])   # subnormal quantum below the normal range
    quantum = Fraction(2) ** (e - bits + 1)
    n, r = divmod(q, quantum)
    if r * 2 > quantum or (r * 2 == quantum and n % 2 == 1):
        n += 1
    return float(n * quantum)


def u8_values(mode) -> np.ndarray:
    """Reading R14: the value of byte u is u / 255 rounded once, to nearest-even, to the latent
    format ('fp16', 'bf16'; 'f32' for the fp32 validation mode).  Returns the 256 values (fp64)."""
    from fractions import Fraction
    return np.array([_round_fraction(Fraction(u, 255), mode) for u in range(256)])


def frames_from_u8(U, mode) -> np.ndarray:
    """8-bit HWC frames U [T,H,W,3] -> NCHW frame values [T,3,H,W] (R14; S:366 to_latent on decoded
    8-bit frames)."""
    U = np.asarray(U, dtype=np.uint8)
    return u8_values(mode)[U].transpose(0, 3, 1, 2).copy()


# --------------------------------------------------------------------------
# conv / norm / activation / resize primitives (R2-R4, R11)
# --------------------------------------------------------------------------
def conv2d(X, Wt, b=None, stride: int = 1, pad: int | None = None):
    """X [T,H,W,Cin], Wt OHWI [Cout,k,k,Cin], b [Cout] -> [T,Ho,Wo,Cout]; zero padding."""
    X, Wt = _f64(X), _f64(Wt)
    T, H, W, Cin = X.shape
    Cout, k, k2, Cin2 = Wt.shape
    if k != k2 or Cin != Cin2:
        raise ValueError("shape mismatch (S:47)")
    if pad is None:
        pad = k // 2
    Ho, Wo = (H + 2 * pad - k) // stride + 1, (W + 2 * pad - k) // stride + 1
    Y = np.empty((T, Ho, Wo, Cout))
    bp = None
    if b is not None:
        b = _f64(b)
        bp = _p(b)
    lib().orc_conv2d(_p(X), T, H, W, Cin, _p(Wt), bp, Cout, k, stride, pad, _p(Y))
    return Y


def conv1x1(X, Wt, b=None):
    """1x1 conv with Wt [Cout,Cin]."""
    Wt = _f64(Wt)
    return conv2d(X, Wt.reshape(Wt.shape[0], 1, 1, Wt.shape[1]), b, 1, 0)


def groupnorm(X, G: int, gamma, beta, eps: float = 1e-5):
    """Per-(frame, group) GroupNorm, biased two-pass variance (R3, R4)."""
    X = _f64(X)
    T = X.shape[0]
    C = X.shape[-1]
    HW = int(np.prod(X.shape[1:-1]))
    if C % G:
        raise ValueError("divisibility error: G must divide C")
    Y = np.empty_like(X)
    g, bt = _f64(gamma), _f64(beta)
    assert lib().orc_groupnorm(_p(X), T, HW, C, G, _p(g), _p(bt), float(eps), _p(Y)) == 0
    return Y


def silu(X):
    X = _f64(X)
    Y = np.empty_like(X)
    lib().orc_silu(_p(X), X.size, _p(Y))
    return Y


def nearest_to(V, Ho: int, Wo: int):
    """U[t,y,x] = V[t, floor(y*H/Ho), floor(x*W/Wo)] (R11)."""
    V = _f64(V)
    T, H, W, C = V.shape
    U = np.empty((T, Ho, Wo, C))
    lib().orc_nearest_to(_p(V), T, H, W, C, Ho, Wo, _p(U))
    return U


# --------------------------------------------------------------------------
# a2. Latent Channel Expansion, encoder side (reading R13)
# --------------------------------------------------------------------------
def expand(L, Wexp, bexp, mode=None):
    """E[t,y,x,k] = b_k + sum_m W[k,m] L[t,y,x,m]; stored 16-bit in 16-bit modes."""
    return rnd(conv1x1(L, Wexp, bexp), mode)


def encode(F, Wexp, bexp, s: int = 8, mode=None):
    """a1 + a2: frames [T,3,H,W] -> expanded latent [T,H/s,W/s,c_lat]."""
    return expand(unshuffle(F, s), Wexp, bexp, mode)


# --------------------------------------------------------------------------
# a3. Temporal shift: batch form and online form
# --------------------------------------------------------------------------
def _check_p(C, P):
    if P < 1 or C % P:
        raise ValueError("divisibility error: P must divide C (S:228)")
    return C // P


def shift_batch(X, carry, P: int):
    """Batch-dimension OTSM: for c < C/P, frame t receives frame t-1's
    channel c (intra-batch); frame 0 receives ``carry`` (inter-batch); the
    rest is unchanged.  carry=None means zeros (chain start, R8).
    Returns (X_shifted, carry_out = X[T-1][..., :C/P])."""
    X = _f64(X)
    c = _check_p(X.shape[-1], P)
    Y = X.copy()
    Y[1:, ..., :c] = X[:-1, ..., :c]
    Y[0, ..., :c] = 0.0 if carry is None else _f64(carry)
    return Y, X[-1, ..., :c].copy()


def shift_online(x_t, state, P: int):
    """Online TSM with a per-layer buffer ("the first segment is cached
    ... the remaining segment is concatenated with the buffered feature slice";
    S:215-218).  x_t [h,w,C]; state [h,w,C/P] or None (zeros at sequence start).
    Returns (y_t, state')."""
    x_t = _f64(x_t)
    C = x_t.shape[-1]
    c = _check_p(C, P)
    cached = np.zeros(x_t.shape[:-1] + (c,)) if state is None else _f64(state)
    y = np.concatenate([cached, x_t[..., c:]], axis=-1)   # buffered slice ++ remaining segment
    return y, x_t[..., :c].copy()                          # first segment cached for frame t+1


# --------------------------------------------------------------------------
# a3-a8. One OTSM ResBlock over T consecutive frames (R2, R5-R8, R15)
# --------------------------------------------------------------------------
def resblock(X, carry, w: dict, G: int, P: int, eps: float = 1e-5, mode=None,
             shift: str = "batch"):
    """Out = S(X) + conv2(silu(gn2(conv1(silu(gn1(shift(X, carry))))))).

    X [T,h,w,Cin]; carry [h,w,Cin/P] or None.  w holds gn1_w, gn1_b, conv1_w,
    conv1_b, gn2_w, gn2_b, conv2_w, conv2_b and, iff Cin != Cout, sc_w [Cout,Cin],
    sc_b.  The shift sits at the entry of the residual branch (R5); the shortcut
    sees the unshifted X.  mode rounds at the storage points H1, Y1, H2, Out
    (R15).  shift='online' runs the shift frame by frame with a buffer instead of
    the batch formula (the two must agree exactly).
    Returns (Out, carry_out)."""
    X = _f64(X)
    if shift == "batch":
        Xs, k_out = shift_batch(X, carry, P)
    else:
        frames, st = [], carry
        for t in range(X.shape[0]):
            y, st = shift_online(X[t], st, P)
            frames.append(y)
        Xs, k_out = np.stack(frames), st
    H1 = rnd(silu(groupnorm(Xs, G, w["gn1_w"], w["gn1_b"], eps)), mode)
    Y1 = rnd(conv2d(H1, w["conv1_w"], w["conv1_b"]), mode)
    H2 = rnd(silu(groupnorm(Y1, G, w["gn2_w"], w["gn2_b"], eps)), mode)
    Y2 = conv2d(H2, w["conv2_w"], w["conv2_b"])
    S = X if w.get("sc_w") is None else conv1x1(X, w["sc_w"], w["sc_b"])
    return rnd(S + Y2, mode), k_out


# --------------------------------------------------------------------------
# f1. Self-attention Transformer2D blocks ("U-Net"; P:525 parameter count;
# readings R24-R27 in DESIGN.md section 3).  SD-2.1's Transformer2DModel with
# the text cross-attention removed: GN -> proj_in -> [LN -> self-attention ->
# +res] -> [LN -> GEGLU FF -> +res] -> proj_out -> + block input.
# --------------------------------------------------------------------------
def layernorm(X, gamma, beta, eps: float = 1e-5):
    """LayerNorm over the channels of every pixel, biased two-pass variance (R24)."""
    X = _f64(X)
    mu = X.mean(axis=-1, keepdims=True)
    var = ((X - mu) ** 2).mean(axis=-1, keepdims=True)
    return (X - mu) / np.sqrt(var + eps) * _f64(gamma) + _f64(beta)


def gelu(X):
    """Exact GELU x * Phi(x) = x/2 * (1 + erf(x / sqrt 2)) (GEGLU gate, R24)."""
    from scipy.special import erf
    X = _f64(X)
    return 0.5 * X * (1.0 + erf(X / np.sqrt(2.0)))


def attention(Q, K, V, head_dim: int, rows=None):
    """Multi-head self-attention of every frame over its own h*w tokens (R25):
    for each frame t and head j (channels [j*d, (j+1)*d)),
        O_j = softmax(Q_j K_j^T / sqrt(d)) V_j   (row softmax).
    Q, K, V [T,N,C]; rows: optional query indices (sampled check at large N).
    Returns [T,N,C] (or [T,len(rows),C])."""
    Q, K, V = _f64(Q), _f64(K), _f64(V)
    T, N, C = Q.shape
    if C % head_dim:
        raise ValueError("divisibility error: head_dim must divide C")
    if rows is not None:
        Q = Q[:, rows]
    O = np.empty_like(Q)
    d = head_dim
    for t in range(T):
        for j in range(C // d):
            sl = slice(j * d, (j + 1) * d)
            S = Q[t, :, sl] @ K[t, :, sl].T / np.sqrt(d)
            S = S - S.max(axis=1, keepdims=True)
            Pm = np.exp(S)
            Pm = Pm / Pm.sum(axis=1, keepdims=True)
            O[t, :, sl] = Pm @ V[t, :, sl]
    return O


TF_ORDER = ("gn_w", "gn_b", "proj_in_w", "proj_in_b", "ln1_w", "ln1_b", "qkv_w", "out_w", "out_b",
            "ln2_w", "ln2_b", "ff1_w", "ff1_b", "ff2_w", "ff2_b", "proj_out_w", "proj_out_b")


def tf_shapes(C: int) -> dict:
    """Tensor shapes of one Transformer2D block of width C (blob order TF_ORDER)."""
    return {"gn_w": (C,), "gn_b": (C,), "proj_in_w": (C, C), "proj_in_b": (C,),
            "ln1_w": (C,), "ln1_b": (C,), "qkv_w": (3 * C, C), "out_w": (C, C), "out_b": (C,),
            "ln2_w": (C,), "ln2_b": (C,), "ff1_w": (8 * C, C), "ff1_b": (8 * C,),
            "ff2_w": (C, 4 * C), "ff2_b": (C,), "proj_out_w": (C, C), "proj_out_b": (C,)}


def transformer(X, w: dict, G: int, head_dim: int, eps_gn: float = 1e-6, eps_ln: float = 1e-5,
                mode=None):
    """One Transformer2D block over X [T,h,w,C] (R24-R27), frames independent:
        a  = GN(X)                          (G groups, eps 1e-6, no SiLU)
        h0 = proj_in(a)                     (1x1, C -> C, bias)
        q,k,v = split(LN1(h0) W_qkv^T)      (no bias)
        h1 = out(attention(q, k, v)) + h0   (1x1 + bias)
        f  = ff1(LN2(h1))                   (C -> 8C, bias); g = f[:4C] * gelu(f[4C:])
        h2 = ff2(g) + h1                    (4C -> C, bias)
        Y  = proj_out(h2) + X               (1x1 + bias)
    mode rounds every stored tensor to 16-bit (R27)."""
    X = _f64(X)
    T, H, W, C = X.shape
    N = H * W
    a = rnd(groupnorm(X, G, w["gn_w"], w["gn_b"], eps_gn), mode)
    h0 = rnd(conv1x1(a, w["proj_in_w"], w["proj_in_b"]), mode)
    l1 = rnd(layernorm(h0, w["ln1_w"], w["ln1_b"], eps_ln), mode)
    qkv = rnd(conv1x1(l1, w["qkv_w"]), mode).reshape(T, N, 3 * C)
    o = rnd(attention(qkv[..., :C], qkv[..., C:2 * C], qkv[..., 2 * C:], head_dim), mode)
    h1 = rnd(conv1x1(o.reshape(T, H, W, C), w["out_w"], w["out_b"]) + h0, mode)
    l2 = rnd(layernorm(h1, w["ln2_w"], w["ln2_b"], eps_ln), mode)
    f = rnd(conv1x1(l2, w["ff1_w"], w["ff1_b"]), mode)
    g = rnd(f[..., :4 * C] * gelu(f[..., 4 * C:]), mode)
    h2 = rnd(conv1x1(g, w["ff2_w"], w["ff2_b"]) + h1, mode)
    return rnd(conv1x1(h2, w["proj_out_w"], w["proj_out_b"]) + X, mode)


# --------------------------------------------------------------------------
# a9-a10. The pruned U-Net ResBlock skeleton (R1, R9-R11)
# --------------------------------------------------------------------------
def unet_blocks(width=(240, 480, 960, 960)):
    """The oracle's own statement of reading R1 (SD-2.1-base U-Net, widths x0.75,
    layers_per_block 2, 22 ResBlocks).  Returns [(name, level, cin, cout)] in
    execution order; up-block cin counts the concatenated skip."""
    blocks = []
    skips = [width[0]]                           # conv_in output
    cur = width[0]
    for l in range(4):
        for r in range(2):
            blocks.append((f"down{l}.r{r}", l, cur, width[l]))
            cur = width[l]
            skips.append(cur)
        if l < 3:
            skips.append(cur)                    # stride-2 downsampler output
    for r in range(2):
        blocks.append((f"mid.r{r}", 3, cur, cur))
    for u in range(4):
        l = 3 - u
        for r in range(3):
            sk = skips.pop()
            blocks.append((f"up{u}.r{r}", l, cur + sk, width[l]))
            cur = width[l]
    return blocks


def param_count(width=(240, 480, 960, 960), c_in=512, c_out=256, attention=True):
    """Closed-form parameter count of reading R1, used to pin it to Table 8's
    444.78 M.  Transformer2D blocks (cross-attention removed) count
    18C^2 + 18C each: GN 2C, proj_in/out 2(C^2+C), LN1 2C, qkv 3C^2, out C^2+C,
    LN 2C, GEGLU C->8C (8C^2+8C), FF out 4C->C (4C^2+C)."""
    n = 9 * c_in * width[0] + width[0]
    for _, _, ci, co in unet_blocks(width):
        n += 9 * ci * co + co + 9 * co * co + co + 2 * ci + 2 * co
        if ci != co:
            n += ci * co + co
    for C in (width[0], width[1], width[2]):           # 3 downsamplers
        n += 9 * C * C + C
    for C in (width[3], width[2], width[1]):           # 3 upsamplers
        n += 9 * C * C + C
    n += 2 * width[0] + 9 * width[0] * c_out + c_out   # norm_out + conv_out
    if attention:
        tb = lambda C: 18 * C * C + 18 * C  # noqa: E731
        n += 2 * (tb(width[0]) + tb(width[1]) + tb(width[2]))   # down 0..2
        n += tb(width[3])                                      # mid
        n += 3 * (tb(width[2]) + tb(width[1]) + tb(width[0]))   # up 1..3
    return n


def _take(it, shape, name):
    nm, a = next(it)
    a = _f64(a)
    if tuple(a.shape) != tuple(shape):
        raise ValueError(f"weight {nm} has shape {a.shape}, oracle expected {name} {shape}")
    return a


def _rb_weights(it, cin, cout):
    w = {
        "gn1_w": _take(it, (cin,), "gn1_w"), "gn1_b": _take(it, (cin,), "gn1_b"),
        "conv1_w": _take(it, (cout, 3, 3, cin), "conv1_w"), "conv1_b": _take(it, (cout,), "conv1_b"),
        "gn2_w": _take(it, (cout,), "gn2_w"), "gn2_b": _take(it, (cout,), "gn2_b"),
        "conv2_w": _take(it, (cout, 3, 3, cout), "conv2_w"), "conv2_b": _take(it, (cout,), "conv2_b"),
        "sc_w": None, "sc_b": None,
    }
    if cin != cout:
        w["sc_w"] = _take(it, (cout, cin), "sc_w")
        w["sc_b"] = _take(it, (cout,), "sc_b")
    return w


def _tf_weights(it, C):
    sh = tf_shapes(C)
    return {k: _take(it, sh[k], k) for k in TF_ORDER}


def skeleton(lat, ctx, weights, width=(240, 480, 960, 960), G: int = 24, P: int = 8,
             eps: float = 1e-5, carries=None, mode=None, record=None, shift="batch", halo=None,
             attention: bool = False, head_dim: int = 48):
    """The pruned U-Net's ResBlock skeleton over T frames of one chain (R1, R11):
        x0 = conv_in(concat(Lbar, Cm));  push x0
        for level l = 0..3: two ResBlocks (push each); if l < 3: conv3x3 stride 2 (push)
        mid: two ResBlocks
        for u = 0..3 (level 3-u): three ResBlocks on concat(h, pop());
                                  if u < 3: nearest to the next skip's size, conv3x3
        out = conv_out(silu(gn_out(h)))
    attention=False: the 16 self-attention Transformer2D blocks are elided (identity).
    attention=True (f1, full U-Net, R26): a Transformer2D block follows every ResBlock of
    down levels 0-2, mid.r0, and every ResBlock of up levels 2-0; its weights follow that
    ResBlock's in the blob (TF_ORDER).
    weights: iterable of (name, array) in the blob order of include/dvc.h.
    carries: list of 22 slices [h_l, w_l, Cin_k/P] (None = chain start, zeros).
    record: optional list that receives every ResBlock output.
    halo: optional callable (k, X) -> carry for block k, called right before block k
    with its input X (multi-GPU lockstep: send X's last-frame slice onward, receive the
    predecessor's); overrides carries[k].
    Returns (out [T,h,w,c_out], carries_out)."""
    it = iter(weights)
    lat, ctx = _f64(lat), _f64(ctx)
    c_cat = lat.shape[-1] + ctx.shape[-1]
    blocks = unet_blocks(width)
    if carries is None:
        carries = [None] * len(blocks)
    k_out = []
    bi = 0

    def run_tf(h):
        if not attention:
            return h
        return transformer(h, _tf_weights(it, h.shape[-1]), G, head_dim, mode=mode)

    def run_block(h):
        nonlocal bi
        name, _, cin, cout = blocks[bi]
        if h.shape[-1] != cin:
            raise ValueError(f"{name}: input has {h.shape[-1]} channels, expected {cin}")
        w = _rb_weights(it, cin, cout)
        carry = halo(bi, h) if halo is not None else carries[bi]
        out, k = resblock(h, carry, w, G, P, eps, mode, shift)
        k_out.append(k)
        if record is not None:
            record.append(out)
        bi += 1
        return out

    w_in = _take(it, (width[0], 3, 3, c_cat), "conv_in_w")
    b_in = _take(it, (width[0],), "conv_in_b")
    h = rnd(conv2d(np.concatenate([lat, ctx], axis=-1), w_in, b_in), mode)
    skips = [h]
    for l in range(4):
        for _ in range(2):
            h = run_block(h)
            if l < 3:
                h = run_tf(h)
            skips.append(h)
        if l < 3:
            C = h.shape[-1]
            wd = _take(it, (C, 3, 3, C), "down_w")
            bd = _take(it, (C,), "down_b")
            h = rnd(conv2d(h, wd, bd, stride=2, pad=1), mode)
            skips.append(h)
    for r in range(2):
        h = run_block(h)
        if r == 0:
            h = run_tf(h)
    for u in range(4):
        for _ in range(3):
            h = run_block(np.concatenate([h, skips.pop()], axis=-1))
            if u > 0:
                h = run_tf(h)
        if u < 3:
            C = h.shape[-1]
            Ho, Wo = skips[-1].shape[1], skips[-1].shape[2]
            wu = _take(it, (C, 3, 3, C), "up_w")
            bu = _take(it, (C,), "up_b")
            h = rnd(conv2d(nearest_to(h, Ho, Wo), wu, bu), mode)
    C = h.shape[-1]
    g_o = _take(it, (C,), "gn_out_w")
    b_o = _take(it, (C,), "gn_out_b")
    c_out = lat.shape[-1]
    w_o = _take(it, (c_out, 3, 3, C), "conv_out_w")
    bo = _take(it, (c_out,), "conv_out_b")
    hn = rnd(silu(groupnorm(h, G, g_o, b_o, eps)), mode)
    out = rnd(conv2d(hn, w_o, bo), mode)
    rest = list(it)
    if rest:
        raise ValueError(f"{len(rest)} unused weight tensors")
    return out, k_out


# --------------------------------------------------------------------------
# f2. Pruned VAE Decoder ("Pruned VAE Decoder reduces intermediate channels by
# 50%", P:108 latent interface expanded to 256 channels; Table 8; readings R29-R31).
# SD-2.1's AutoencoderKL decoder with block widths x0.5 = (64, 128, 256, 256), no temporal
# shift (frames independent).
# --------------------------------------------------------------------------
def vae_resblock(X, w: dict, G: int, eps: float, mode=None):
    """SD VAE ResnetBlock2D: Out = S(X) + conv2(silu(gn2(conv1(silu(gn1(X)))))) (no shift)."""
    X = _f64(X)
    H1 = rnd(silu(groupnorm(X, G, w["gn1_w"], w["gn1_b"], eps)), mode)
    Y1 = rnd(conv2d(H1, w["conv1_w"], w["conv1_b"]), mode)
    H2 = rnd(silu(groupnorm(Y1, G, w["gn2_w"], w["gn2_b"], eps)), mode)
    Y2 = conv2d(H2, w["conv2_w"], w["conv2_b"])
    S = X if w.get("sc_w") is None else conv1x1(X, w["sc_w"], w["sc_b"])
    return rnd(S + Y2, mode)


def vae_attention(X, w: dict, G: int, eps: float, mode=None):
    """SD VAE mid-block attention: single head over the h*w tokens of each frame,
    Y = X + out(softmax(q k^T / sqrt C) v), q/k/v/out linear with bias on GN(X)."""
    X = _f64(X)
    T, H, W, C = X.shape
    a = rnd(groupnorm(X, G, w["gn_w"], w["gn_b"], eps), mode)
    q = rnd(conv1x1(a, w["q_w"], w["q_b"]), mode).reshape(T, H * W, C)
    k = rnd(conv1x1(a, w["k_w"], w["k_b"]), mode).reshape(T, H * W, C)
    v = rnd(conv1x1(a, w["v_w"], w["v_b"]), mode).reshape(T, H * W, C)
    o = rnd(attention(q, k, v, C), mode).reshape(T, H, W, C)
    return rnd(conv1x1(o, w["out_w"], w["out_b"]) + X, mode)


def vae_blocks(width=(64, 128, 256, 256)):
    """Reading R29: [(name, level, cin, cout)] of the decoder's ResBlocks in execution order;
    level 0 = latent resolution, 3 = full resolution."""
    top = width[-1]
    blocks = [("mid.r0", 0, top, top), ("mid.r1", 0, top, top)]
    cur = top
    for i, c in enumerate(reversed(width)):
        for r in range(3):
            blocks.append((f"up{i}.r{r}", i, cur, c))
            cur = c
    return blocks


def vae_param_count(width=(64, 128, 256, 256), c_lat=256, out_ch=3, mid_attn=True):
    """Closed form of reading R29 (compare Table 8: 12.38 M)."""
    top = width[-1]
    n = 9 * c_lat * top + top
    for _, _, ci, co in vae_blocks(width):
        n += 2 * ci + 9 * ci * co + co + 2 * co + 9 * co * co + co + (ci * co + co if ci != co else 0)
    if mid_attn:
        n += 2 * top + 4 * (top * top + top)
    for c in list(reversed(width))[:3]:
        n += 9 * c * c + c
    return n + 2 * width[0] + 9 * width[0] * out_ch + out_ch


def vae_decode(L, weights, width=(64, 128, 256, 256), G: int = 32, eps: float = 1e-6, out_ch: int = 3,
               mid_attn: bool = True, mode=None):
    """L [T,h,w,c_lat] (the U-Net's Lhat) -> frames [T,8h,8w,out_ch] (NHWC), R29-R31:
        x = conv_in(L); mid: ResBlock, [attention], ResBlock
        for i = 0..3 (widths reversed): 3 ResBlocks; if i < 3: nearest 2x, conv3x3
        out = conv_out(silu(gn_out(x)))
    weights: iterable of (name, array) in the blob order of include/dvc.h (dvc_vae_create)."""
    it = iter(weights)
    L = _f64(L)
    top = width[-1]
    x = rnd(conv2d(L, _take(it, (top, 3, 3, L.shape[-1]), "conv_in_w"), _take(it, (top,), "conv_in_b")), mode)
    blocks = vae_blocks(width)
    bi = 0

    def rb(x):
        nonlocal bi
        _, _, ci, co = blocks[bi]
        bi += 1
        return vae_resblock(x, _rb_weights(it, ci, co), G, eps, mode)

    x = rb(x)
    if mid_attn:
        sh = {"gn_w": (top,), "gn_b": (top,), "q_w": (top, top), "q_b": (top,), "k_w": (top, top), "k_b": (top,),
              "v_w": (top, top), "v_b": (top,), "out_w": (top, top), "out_b": (top,)}
        x = vae_attention(x, {k: _take(it, sh[k], k) for k in sh}, G, eps, mode)
    x = rb(x)
    for i, c in enumerate(reversed(width)):
        for _ in range(3):
            x = rb(x)
        if i < 3:
            T, H, W, _ = x.shape
            x = rnd(conv2d(nearest_to(x, 2 * H, 2 * W), _take(it, (c, 3, 3, c), "up_w"), _take(it, (c,), "up_b")),
                    mode)
    C = x.shape[-1]
    g, b = _take(it, (C,), "gn_out_w"), _take(it, (C,), "gn_out_b")
    hn = rnd(silu(groupnorm(x, G, g, b, eps)), mode)
    out = rnd(conv2d(hn, _take(it, (out_ch, 3, 3, C), "conv_out_w"), _take(it, (out_ch,), "conv_out_b")), mode)
    rest = list(it)
    if rest:
        raise ValueError(f"{len(rest)} unused weight tensors")
    return out


# --------------------------------------------------------------------------
# f4 variant: fp8 E4M3 quantisation (OCP FP8 E4M3 "fn": bias 7, 3 mantissa bits, no
# infinities, max 448, subnormal quantum 2^-9) and the dequantised convolution
# --------------------------------------------------------------------------
def e4m3_round(v):
    """Round-to-nearest-even to E4M3, saturating to +-448 (the GPU's SATFINITE conversion).
    v: fp64 array of the values to round (callers pass the fp32 quotient x / scale)."""
    v = _f64(v)
    a = np.abs(v)
    fin = np.isfinite(a)
    af = np.where(fin, a, 0.0)
    e = np.floor(np.log2(np.where(af > 0, af, 1.0)))
    e = np.maximum(e, -6.0)                        # below 2^-6: subnormal quantum 2^-9
    q = np.exp2(e - 3.0)
    r = np.round(af / q) * q                       # numpy rounds half to even; af / q is exact
    r = np.where(fin, np.minimum(r, 448.0), 448.0)  # saturating: +-inf and overflow -> +-448
    return np.where(np.isnan(v), np.nan, np.sign(v) * r)


def quantize_e4m3(x, scale: float):
    """q = E4M3(x / scale), the quotient taken in fp32 as the GPU does (R32)."""
    quot = (np.asarray(x, np.float32) / np.float32(scale)).astype(np.float64)
    return e4m3_round(quot)


def conv_fp8(q_x, sx: float, q_w, sw: float, b=None):
    """The fp8 convolution's exact value: conv(sx * q_x, sw * q_w) + b in fp64 (3x3 pad 1 or 1x1)."""
    k = q_w.shape[1]
    return conv2d(_f64(q_x) * sx, _f64(q_w) * sw, b, 1, k // 2)


def rel_l2(a, ref) -> float:
    """||a - ref||_2 / ||ref||_2 (R16)."""
    a, ref = _f64(a), _f64(ref)
    return float(np.linalg.norm((a - ref).ravel()) / max(np.linalg.norm(ref.ravel()), 1e-300))
