"""Pins of the fp64 oracle to things other than itself (-m "not gpu").

Each test ties an oracle routine to what the paper / mathematics fix: SPEC
worked examples (S:<line>), closed forms, special cases that reduce to a
library routine (torch CPU fp64), brute force on tiny inputs, invariants.
"""
import itertools
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synthgen

RTOL = 1e-12


def _nchw(x):
    return torch.from_numpy(np.ascontiguousarray(x)).permute(0, 3, 1, 2)


def _nhwc(t):
    return t.permute(0, 2, 3, 1).contiguous().numpy()


# ---------------------------------------------------------------- a1 unshuffle
def test_unshuffle_shape_example(orc):          # S:59 (1,3,8,8), s=8 -> (1,192,1,1)
    x = np.arange(192, dtype=np.float64).reshape(1, 3, 8, 8)
    L = orc.unshuffle(x, 8)
    assert L.shape == (1, 1, 1, 192)
    # channel c*64 + i*8 + j holds F[c, i, j]  (torch order, R12) -> here 0..191 in order
    assert np.array_equal(L.ravel(), np.arange(192))


def test_unshuffle_s1_identity(orc):
    x = np.random.default_rng(0).standard_normal((2, 3, 4, 6))
    assert np.array_equal(orc.unshuffle(x, 1), x.transpose(0, 2, 3, 1))


@pytest.mark.parametrize("s,H,W", [(8, 16, 24), (2, 6, 4), (4, 8, 12)])
def test_unshuffle_vs_torch_and_roundtrip(orc, s, H, W):
    x = np.random.default_rng(s).standard_normal((3, 3, H, W))
    L = orc.unshuffle(x, s)
    ref = F.pixel_unshuffle(torch.from_numpy(x), s)
    assert np.array_equal(L, _nhwc(ref))
    assert np.array_equal(orc.shuffle(L, 3, s), x)


def test_unshuffle_divisibility(orc):
    with pytest.raises(ValueError):
        orc.unshuffle(np.zeros((1, 3, 12, 16)), 8)


# ---------------------------------------------------------------- a2 expansion
def test_expansion_identity_weights(orc):
    L = np.random.default_rng(1).standard_normal((2, 3, 5, 192))
    W = np.concatenate([np.eye(192), np.zeros((64, 192))])
    E = orc.expand(L, W, np.zeros(256))
    assert np.array_equal(E[..., :192], L) and not E[..., 192:].any()


def test_expansion_vs_matmul(orc):
    g = np.random.default_rng(2)
    L, W, b = g.standard_normal((2, 3, 4, 192)), g.standard_normal((256, 192)), g.standard_normal(256)
    ref = np.einsum("thwm,km->thwk", L, W) + b
    np.testing.assert_allclose(orc.expand(L, W, b), ref, rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- conv (a5, a7, a9)
def test_conv_identity_kernel(orc):
    x = np.random.default_rng(3).standard_normal((2, 4, 5, 6))
    w = np.zeros((6, 3, 3, 6))
    w[:, 1, 1, :] = np.eye(6)
    assert np.array_equal(orc.conv2d(x, w, np.zeros(6)), x)
    assert np.array_equal(orc.conv1x1(x, np.eye(6)), x)


def test_conv_all_ones(orc):
    y = orc.conv2d(np.ones((1, 5, 5, 1)), np.ones((1, 3, 3, 1)), None)[0, ..., 0]
    assert y[2, 2] == 9 and y[0, 2] == 6 and y[2, 0] == 6 and y[0, 0] == 4 and y[4, 4] == 4


def test_conv_brute_force(orc):                 # S:52, random 2x3x4x4
    g = np.random.default_rng(4)
    x, w, b = g.standard_normal((2, 4, 4, 3)), g.standard_normal((5, 3, 3, 3)), g.standard_normal(5)
    y = orc.conv2d(x, w, b)
    ref = np.zeros((2, 4, 4, 5))
    for t, oy, ox, o in itertools.product(range(2), range(4), range(4), range(5)):
        s = b[o]
        for ky, kx, c in itertools.product(range(3), range(3), range(3)):
            iy, ix = oy + ky - 1, ox + kx - 1
            if 0 <= iy < 4 and 0 <= ix < 4:
                s += w[o, ky, kx, c] * x[t, iy, ix, c]
        ref[t, oy, ox, o] = s
    np.testing.assert_allclose(y, ref, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("stride,H,W", [(1, 7, 9), (2, 7, 9), (2, 8, 10), (1, 3, 3)])
def test_conv_vs_torch(orc, stride, H, W):
    g = np.random.default_rng(5)
    x, w, b = g.standard_normal((2, H, W, 8)), g.standard_normal((6, 3, 3, 8)), g.standard_normal(6)
    y = orc.conv2d(x, w, b, stride=stride, pad=1)
    ref = F.conv2d(_nchw(x), torch.from_numpy(w).permute(0, 3, 1, 2), torch.from_numpy(b),
                   stride=stride, padding=1)
    np.testing.assert_allclose(y, _nhwc(ref), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("H,ref", [(90, [45, 23, 12]), (135, [68, 34, 17]), (160, [80, 40, 20]),
                                   (240, [120, 60, 30])])
def test_stride2_chain_sizes(orc, H, ref):      # SURVEY P12 (ceil halving)
    sizes, h = [], H
    for _ in range(3):
        h = orc.conv2d(np.zeros((1, h, 1, 1)), np.zeros((1, 3, 3, 1)), None, 2, 1).shape[1]
        sizes.append(h)
    assert sizes == ref


# ---------------------------------------------------------------- GN + SiLU (a4, a6)
def test_groupnorm_constant_group_gives_beta(orc):
    x = np.full((2, 3, 4, 8), 1.75)
    beta = np.linspace(-0.5, 0.5, 8)
    y = orc.groupnorm(x, 4, np.full(8, 1.3), beta)
    assert np.array_equal(y, np.broadcast_to(beta, y.shape))


def test_groupnorm_two_value_closed_form(orc):
    # one group, half the entries a and half b: mu=(a+b)/2, var=((a-b)/2)^2
    a, b, eps = 3.0, -1.0, 1e-5
    x = np.empty((1, 2, 2, 2))
    x[..., 0], x[..., 1] = a, b
    y = orc.groupnorm(x, 1, np.ones(2), np.zeros(2), eps)
    d = (a - b) / 2 / math.sqrt(((a - b) / 2) ** 2 + eps)
    np.testing.assert_allclose(y[..., 0], d, rtol=1e-15)
    np.testing.assert_allclose(y[..., 1], -d, rtol=1e-15)


@pytest.mark.parametrize("C,G", [(240, 24), (64, 32), (48, 8)])
def test_groupnorm_vs_torch(orc, C, G):
    g = np.random.default_rng(6)
    x = g.standard_normal((3, 5, 7, C)) * 2 + 0.5
    gam, bet = g.uniform(0.5, 1.5, C), g.uniform(-0.5, 0.5, C)
    y = orc.groupnorm(x, G, gam, bet, 1e-5)
    ref = F.group_norm(_nchw(x), G, torch.from_numpy(gam), torch.from_numpy(bet), 1e-5)
    np.testing.assert_allclose(y, _nhwc(ref), rtol=1e-10, atol=1e-10)


def test_silu(orc):                             # S:78 silu(0) = 0
    assert orc.silu(np.zeros(3)).tolist() == [0.0, 0.0, 0.0]
    x = np.linspace(-30, 30, 1001)
    np.testing.assert_allclose(orc.silu(x), F.silu(torch.from_numpy(x)).numpy(), rtol=1e-14, atol=1e-300)


# ---------------------------------------------------------------- nearest to size (a9)
@pytest.mark.parametrize("hi,ho", [(12, 23), (23, 45), (45, 90), (17, 34), (34, 68), (68, 135), (20, 40),
                                   (3, 7), (5, 5)])
def test_nearest_to_vs_torch(orc, hi, ho):
    v = np.random.default_rng(hi).standard_normal((2, hi, hi + 1, 3))
    u = orc.nearest_to(v, ho, ho + 2)
    ref = F.interpolate(_nchw(v), size=(ho, ho + 2), mode="nearest")
    assert np.array_equal(u, _nhwc(ref))


@pytest.mark.parametrize("h,w", [(12, 20), (23, 40), (68, 120), (2, 3), (9, 14), (1, 1)])
def test_nearest_to_2h_minus_1_is_clipped_phase_replication(orc, h, w):
    # the identity the GPU upsampler folds rely on (DESIGN §2 / §10): R11's nearest_to onto
    # 2H or 2H - 1 rows (2W or 2W - 1 columns) is the exact 2x replication cropped at the far edge
    v = np.random.default_rng(h * 100 + w).standard_normal((2, h, w, 3))
    rep = np.repeat(np.repeat(v, 2, axis=1), 2, axis=2)
    for ho in (2 * h - 1, 2 * h):
        for wo in (2 * w - 1, 2 * w):
            if ho < 1 or wo < 1:
                continue
            assert np.array_equal(orc.nearest_to(v, ho, wo), rep[:, :ho, :wo])
    # and only there: one more row or one less breaks it (the fold is gated on these two sizes)
    if h >= 2:
        u = orc.nearest_to(v, 2 * h - 2, 2 * w)
        assert not np.array_equal(u, rep[:, :2 * h - 2, :2 * w])


# ---------------------------------------------------------------- rounding (R15)
def test_round_spec_examples(orc):
    assert orc.rnd1(65520.0, "fp16") == math.inf
    assert orc.rnd1(-65520.0, "fp16") == -math.inf
    assert orc.rnd1(65519.99, "fp16") == 65504.0
    assert orc.rnd1(math.pi, "bf16") == 3.140625
    assert orc.rnd1(1.0, "bf16") == 1.0
    assert orc.rnd1(65520.0, "bf16") == 65536.0                       # bf16 has fp32's range
    assert orc.rnd1(1 + 2 ** -8, "bf16") == 1.0                       # tie -> even
    assert orc.rnd1(1 + 3 * 2 ** -8, "bf16") == 1 + 2 ** -6           # tie -> even (up)


def test_round_fp16_exhaustive_vs_numpy(orc):
    # every finite binary16 value, every midpoint between neighbours (ties) and
    # random doubles: numpy's float64->float16 cast is correctly rounded.
    h = np.arange(0, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float64)
    mids = (h[:-1] + h[1:]) / 2
    g = np.random.default_rng(7)
    rand = np.concatenate([g.standard_normal(20000) * 10.0 ** g.integers(-8, 5, 20000)])
    for v in (h, mids, rand, -mids):
        np.testing.assert_array_equal(orc.rnd(v, "fp16"), v.astype(np.float16).astype(np.float64))


def test_round_bf16_vs_torch(orc):
    # fp32-representable inputs: torch's fp32->bf16 cast is RNE (single rounding).
    g = np.random.default_rng(8)
    v = (g.standard_normal(50000) * 10.0 ** g.integers(-30, 30, 50000)).astype(np.float32)
    mids = np.arange(0, 0x7F7F, 7, dtype=np.uint32)
    mids = ((mids << 16) | 0x8000).view(np.float32)                   # exact bf16 midpoints
    for x in (v, mids):
        ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
        np.testing.assert_array_equal(orc.rnd(x.astype(np.float64), "bf16"), ref)


def test_round_double_not_via_fp32(orc):
    # 1 + 2^-8 + 2^-40: just above the bf16 tie -> must round up; rounding via
    # fp32 first would land on the tie and round to even (down).
    assert orc.rnd1(1 + 2 ** -8 + 2 ** -40, "bf16") == 1 + 2 ** -7


def test_round_idempotent(orc):
    x = np.random.default_rng(9).standard_normal(10000) * 100
    for m in ("fp16", "bf16"):
        r = orc.rnd(x, m)
        assert np.array_equal(orc.rnd(r, m), r)


# ---------------------------------------------------------------- a3 temporal shift
def _unique(T, h, w, C):
    return np.arange(T * h * w * C, dtype=np.float64).reshape(T, h, w, C) + 1


def test_shift_is_selection(orc):
    T, C, P = 5, 16, 4
    x = _unique(T, 2, 3, C)
    k = -_unique(1, 2, 3, C // P)[0]
    y, k2 = orc.shift_batch(x, k, P)
    assert np.array_equal(y[0, ..., :4], k)                  # inter-batch shift
    assert np.array_equal(y[1:, ..., :4], x[:-1, ..., :4])  # intra-batch +1 shift
    assert np.array_equal(y[..., 4:], x[..., 4:])           # remaining (P-1)/P untouched
    assert np.array_equal(k2, x[-1, ..., :4])
    vals = set(y.ravel().tolist())
    assert vals <= set(x.ravel().tolist()) | set(k.ravel().tolist())


def test_shift_zero_carry_and_full_shift(orc):
    x = _unique(3, 2, 2, 8)
    y, _ = orc.shift_batch(x, None, 8)
    assert not y[0, ..., :1].any()
    y1, _ = orc.shift_batch(x, None, 1)                      # P=1: previous frame entirely
    assert np.array_equal(y1[1:], x[:-1]) and not y1[0].any()


def test_shift_online_three_frames(orc):         # S:223 P=4, c=8 stacked-array oracle
    x = np.random.default_rng(10).standard_normal((3, 2, 2, 8))
    st, outs = None, []
    for t in range(3):
        y, st = orc.shift_online(x[t], st, 4)
        outs.append(y)
    ref = x.copy()
    ref[:, ..., :2] = np.concatenate([np.zeros((1, 2, 2, 2)), x[:-1, ..., :2]])
    assert np.array_equal(np.stack(outs), ref)


def test_shift_identical_frames(orc):
    x = np.repeat(np.random.default_rng(11).standard_normal((1, 2, 3, 8)), 4, axis=0)
    y, _ = orc.shift_batch(x, None, 4)
    assert not y[0, ..., :2].any() and np.array_equal(y[1:], x[1:])


def _regroup(T, N):
    out, t = [], 0
    while t < T:
        out.append((t, min(T, t + N)))
        t += N
    return out


@pytest.mark.parametrize("P", [2, 4, 8])
def test_batch_equals_online_matrix(orc, P):
    C = 16
    for T in range(1, 13):
        x = np.random.default_rng(T).standard_normal((T, 2, 3, C))
        st, online = None, []
        for t in range(T):
            y, st = orc.shift_online(x[t], st, P)
            online.append(y)
        online = np.stack(online)
        for N in (1, 2, 3, 4, 8):
            carry, parts = None, []
            for a, b in _regroup(T, N):
                y, carry = orc.shift_batch(x[a:b], carry, P)
                parts.append(y)
            assert np.array_equal(np.concatenate(parts), online), (T, N, P)
            assert np.array_equal(carry, st)


def test_shift_causal(orc):
    x = np.random.default_rng(12).standard_normal((6, 2, 2, 8))
    y, _ = orc.shift_batch(x, None, 4)
    x2 = x.copy()
    x2[4:] += 1.0
    y2, _ = orc.shift_batch(x2, None, 4)
    assert np.array_equal(y[:4], y2[:4])


@pytest.mark.parametrize("C,G,ok", [(240, 24, True), (64, 32, True), (240, 16, True), (240, 30, False)])
def test_gn_shift_commutation(orc, C, G, ok):    # holds iff G % P == 0
    g = np.random.default_rng(13)
    x = g.standard_normal((4, 5, 7, C))
    gam, bet = g.uniform(0.5, 1.5, C), g.uniform(-0.5, 0.5, C)
    a = orc.silu(orc.groupnorm(orc.shift_batch(x, None, 8)[0], G, gam, bet))
    b = orc.shift_batch(orc.silu(orc.groupnorm(x, G, gam, bet)), None, 8)[0]
    same = np.allclose(a[1:], b[1:], rtol=1e-13, atol=1e-13)
    assert same == ok
    if ok:   # chain-start slice is SiLU(beta) under R5/R8
        np.testing.assert_allclose(a[0, ..., :C // 8], np.broadcast_to(orc.silu(bet[:C // 8]), (5, 7, C // 8)))


# ---------------------------------------------------------------- a3-a8 ResBlock wiring
def _rb(cin, cout, seed=0):
    return {k: (None if v is None else v.astype(np.float64))
            for k, v in synthgen.resblock_weights(cin, cout, seed).items()}


@pytest.mark.parametrize("cin,cout", [(32, 32), (48, 32)])
def test_resblock_zero_conv2_gives_shortcut(orc, cin, cout):
    w = _rb(cin, cout)
    w["conv2_w"][:] = 0
    w["conv2_b"][:] = 0
    x = np.random.default_rng(14).standard_normal((3, 4, 5, cin))
    out, k = orc.resblock(x, None, w, 8, 8)
    ref = x if cin == cout else orc.conv1x1(x, w["sc_w"], w["sc_b"])   # unshifted X (R5)
    assert np.array_equal(out, ref)
    assert np.array_equal(k, x[-1, ..., :cin // 8])


def test_resblock_shift_isolation(orc):
    cin = cout = 32
    P, G = 8, 8
    x = np.random.default_rng(15).standard_normal((4, 4, 5, cin))
    w = _rb(cin, cout)
    w0 = dict(w)
    w0["conv1_w"] = w["conv1_w"].copy()
    w0["conv1_w"][..., :cin // P] = 0        # slice columns dead -> frame t independent of t-1
    out, _ = orc.resblock(x, None, w0, G, P)
    x2 = x.copy()
    x2[1] += 3.0
    out2, _ = orc.resblock(x2, np.ones((4, 5, cin // P)), w0, G, P)
    assert np.array_equal(out[2:], out2[2:]) and np.array_equal(out[0], out2[0])
    # flipped: only slice columns live -> the residual branch of frame t depends only on frame t-1's
    # slice (the carry for t = 0); the slice is whole GN groups (G % P == 0), so its statistics too
    # (a 1x1 shortcut with zero weights makes Out the residual branch exactly: 0 + Y2 = Y2)
    w1 = _rb(cin, 40)
    w1["sc_w"][:] = 0
    w1["sc_b"][:] = 0
    live = w1["conv1_w"][..., :cin // P].copy()
    w1["conv1_w"][:] = 0
    w1["conv1_w"][..., :cin // P] = live
    r_a, _ = orc.resblock(x, None, w1, G, P)
    x3 = x.copy()
    noise = np.random.default_rng(18).standard_normal(x.shape[1:])   # (a constant shift would be GN-invariant)
    x3[2, ..., cin // P:] += noise[..., cin // P:]   # frame 2 outside the slice: no residual branch moves
    assert np.array_equal(r_a, orc.resblock(x3, None, w1, G, P)[0])
    x4 = x.copy()
    x4[2, ..., :cin // P] += noise[..., :cin // P]   # frame 2's slice: only frame 3's residual branch moves
    r_c, _ = orc.resblock(x4, None, w1, G, P)
    assert np.array_equal(r_a[[0, 1, 2]], r_c[[0, 1, 2]])
    assert np.abs(r_a[3] - r_c[3]).max() > 1e-3
    k = np.random.default_rng(17).standard_normal((4, 5, cin // P))
    r_d, _ = orc.resblock(x, k, w1, G, P)     # the carry: only frame 0's residual branch moves
    assert np.array_equal(r_a[1:], r_d[1:]) and np.abs(r_a[0] - r_d[0]).max() > 1e-3


@pytest.mark.parametrize("cin,cout,T", [(32, 32, 5), (48, 32, 4)])
def test_resblock_batch_equals_online(orc, cin, cout, T):
    w = _rb(cin, cout, 3)
    x = np.random.default_rng(16).standard_normal((T, 3, 4, cin))
    full, kf = orc.resblock(x, None, w, 8, 8)
    online, _ = orc.resblock(x, None, w, 8, 8, shift="online")
    assert np.array_equal(full, online)
    carry, parts = None, []
    for t in range(T):
        y, carry = orc.resblock(x[t:t + 1], carry, w, 8, 8)
        parts.append(y)
    assert np.array_equal(np.concatenate(parts), full) and np.array_equal(carry, kf)


# ---------------------------------------------------------------- a9/a10 topology (R1 pinned by P:525)
def test_param_count_matches_table8(orc):        # 444.776 M vs 444.78 M
    n = orc.param_count()
    assert abs(n / 1e6 - 444.78) < 0.005, n
    for cin in (384, 256, 576):                  # conv_in = concat(Lbar 256, Cm 256) = 512 only
        assert abs(orc.param_count(c_in=cin) / 1e6 - 444.78) > 0.1


def test_topology_block_list(orc):
    blocks = orc.unet_blocks()
    assert len(blocks) == 22                     # P:320 "all 22 ResBlocks"
    cins = [b[2] for b in blocks]
    assert cins == [240, 240, 240, 480, 480, 960, 960, 960, 960, 960,
                    1920, 1920, 1920, 1920, 1920, 1440, 1440, 960, 720, 720, 480, 480]
    assert sum(1 for b in blocks if b[2] != b[3]) == 14     # 1x1 shortcuts


SMALL = (32, 64, 96, 96)


def test_skeleton_batch_equals_online(orc):      # SURVEY P9 for the stack
    T, h, w = 3, 6, 10
    wts = [(n, a.astype(np.float64)) for n, a in synthgen.unet_weights(SMALL, 32, 32)]
    lat, ctx = synthgen.normal((T, h, w, 32), 1), synthgen.normal((T, h, w, 32), 5)
    full, kf = orc.skeleton(lat, ctx, wts, SMALL, G=8, P=8)
    assert full.shape == (T, h, w, 32)
    carries, parts = None, []
    for t in range(T):
        y, carries = orc.skeleton(lat[t:t + 1], ctx[t:t + 1], wts, SMALL, G=8, P=8, carries=carries)
        parts.append(y)
    assert np.array_equal(np.concatenate(parts), full)
    assert all(np.array_equal(a, b) for a, b in zip(carries, kf))
    online, _ = orc.skeleton(lat, ctx, wts, SMALL, G=8, P=8, shift="online")
    assert np.array_equal(online, full)


def test_skeleton_causal(orc):
    T, h, w = 3, 5, 7
    wts = [(n, a.astype(np.float64)) for n, a in synthgen.unet_weights(SMALL, 32, 32)]
    lat, ctx = synthgen.normal((T, h, w, 32), 1), synthgen.normal((T, h, w, 32), 5)
    a, _ = orc.skeleton(lat, ctx, wts, SMALL, G=8, P=8)
    lat2 = lat.copy()
    lat2[2] += 1
    b, _ = orc.skeleton(lat2, ctx, wts, SMALL, G=8, P=8)
    assert np.array_equal(a[:2], b[:2]) and not np.array_equal(a[2], b[2])


# ---------------------------------------------------------------- R14 8-bit frames (G2's reference)
def test_u8_values_closed_forms_and_library(orc):
    for mode in ("fp16", "bf16", "f32"):
        v = orc.u8_values(mode)
        assert v[0] == 0.0 and v[255] == 1.0 and np.all(np.diff(v) >= 0)
        assert np.all(np.abs(v - np.arange(256) / 255.0) <= {"fp16": 2.0 ** -12, "bf16": 2.0 ** -9,
                                                              "f32": 2.0 ** -25}[mode])
    assert np.all(np.diff(orc.u8_values("fp16")) > 0)                      # 11 bits separate all 256
    assert orc.u8_values("fp16")[51] == 0.199951171875                     # RNE_fp16(0.2) (closed form)
    assert orc.u8_values("bf16")[51] == 0.2001953125                       # RNE_bf16(0.2): 0x3E4D
    # independent library roundings of the fp64 quotient agree for all 256 bytes
    q = np.arange(256) / 255.0
    assert np.array_equal(orc.u8_values("fp16"), q.astype(np.float16).astype(np.float64))
    assert np.array_equal(orc.u8_values("f32"), q.astype(np.float32).astype(np.float64))
    assert np.array_equal(orc.u8_values("bf16"), orc.rnd(q, "bf16"))


def test_frames_from_u8_layout(orc):
    U = synthgen.frames_u8_hwc(2, 16, 24)
    F = orc.frames_from_u8(U, "bf16")
    assert F.shape == (2, 3, 16, 24)
    assert np.array_equal(F, orc.rnd(synthgen.frames_u8(2, 16, 24).astype(np.float64) / 255.0, "bf16"))
