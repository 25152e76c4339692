"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle.

Bit-exact for index work (unshuffle, shift, carry); rel-L2 <= 1e-2 for
16-bit outputs against the storage-rounding-emulated oracle (R15/R16) and
<= 1e-5 for the fp32 validation mode against the pure fp64 oracle.
"""
import numpy as np
import pytest
import torch

import synthgen
from tests.gpu_helpers import MODE, TOL, dev, gate, host64, rb_device, rel_l2

pytestmark = pytest.mark.gpu

DTYPES = [torch.bfloat16, torch.float16]


@pytest.fixture(scope="module")
def dvc():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2601_20564_b200 as m
    m.device_check(0)
    return m


# ---------------------------------------------------------------- a1 unshuffle (bit-exact)
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32])
@pytest.mark.parametrize("T,H,W,s", [(1, 8, 8, 8), (3, 24, 40, 8), (2, 16, 136, 8), (2, 12, 20, 4), (1, 6, 6, 2)])
def test_unshuffle_bitexact(dvc, orc, dtype, T, H, W, s):
    f, f64 = dev(synthgen.frames(T, H, W, seed=T + H), dtype)
    out = dvc.dvc_encode_pixelunshuffle(f, s=s)
    torch.cuda.synchronize()
    assert np.array_equal(host64(out), orc.unshuffle(f64, s))


def test_unshuffle_720p_gop_bitexact(dvc, orc):   # config C2 size, bit-exact
    f, f64 = dev(synthgen.frames(32, 720, 1280), torch.float16)
    out = dvc.dvc_encode_pixelunshuffle(f)
    assert np.array_equal(host64(out), orc.unshuffle(f64, 8))


def test_unshuffle_errors(dvc):
    f = torch.zeros((1, 3, 12, 16), dtype=torch.float16, device="cuda")
    with pytest.raises(dvc.DvcError) as e:
        dvc.dvc_encode_pixelunshuffle(f, s=8)
    assert e.value.name == "DVC_ERR_DIVISIBILITY"


# ---------------------------------------------------------------- R14 / G2: 8-bit HWC frames (bit-exact)
def _all_bytes_u8(T, H, W, seed):
    """8-bit HWC frames whose first 256 bytes are every value 0..255 (exhaustive G2), rest random."""
    U = synthgen.frames_u8_hwc(T, H, W, seed)
    flat = U.reshape(-1)
    n = min(256, flat.size)
    flat[:n] = np.arange(n, dtype=np.uint8)
    return U


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32])
@pytest.mark.parametrize("T,H,W,s", [(1, 16, 32, 8), (3, 24, 40, 8), (2, 12, 20, 4), (1, 6, 6, 2)])
def test_unshuffle_u8_bitexact(dvc, orc, dtype, T, H, W, s):
    U = _all_bytes_u8(T, H, W, seed=T + H)
    out = dvc.dvc_encode_pixelunshuffle(torch.from_numpy(U).cuda(), s=s, latent_dtype=dtype)
    ref = orc.unshuffle(orc.frames_from_u8(U, {torch.float32: "f32"}.get(dtype, MODE[dtype])), s)
    assert np.array_equal(host64(out), ref)


def test_u8_conversion_exhaustive(dvc, orc):   # G2: every byte value, each latent type, vs the R14 table
    U = np.zeros((1, 8, 256, 3), dtype=np.uint8)
    U[0, :, :, :] = np.arange(256, dtype=np.uint8)[None, :, None]
    for dtype, mode in ((torch.bfloat16, "bf16"), (torch.float16, "fp16"), (torch.float32, "f32")):
        out = host64(dvc.dvc_encode_pixelunshuffle(torch.from_numpy(U).cuda(), latent_dtype=dtype))
        # latent pixel x covers bytes 8x..8x+7; channel c*64 + i*8 + j holds byte 8x+j of colour c
        got = out[0, 0, :, :8].reshape(-1)
        assert np.array_equal(got, orc.u8_values(mode)), mode


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("T,H,W", [(1, 16, 16), (3, 64, 80), (2, 720, 1280)])
def test_expansion_u8_frames(dvc, orc, dtype, T, H, W):
    """The fused u8 path (converter warps) == the 16-bit NCHW path fed the R14 values, bit for bit;
    and against the oracle within the gates."""
    U = _all_bytes_u8(T, H, W, seed=7)
    w, b = synthgen.expansion_weights()
    wd, w64 = dev(w, dtype)
    bd, b64 = dev(b, dtype)
    out = dvc.dvc_encode_pixelunshuffle(torch.from_numpy(U).cuda(), wd, bd)
    F = orc.frames_from_u8(U, MODE[dtype])
    f16 = torch.from_numpy(F).to(dtype).cuda()
    assert torch.equal(out, dvc.dvc_encode_pixelunshuffle(f16, wd, bd))
    if T * H * W <= 3 * 64 * 80:
        gate(host64(out), orc.encode(F, w64, b64, 8, MODE[dtype]), dtype)


# ---------------------------------------------------------------- a2 expansion
@pytest.mark.parametrize("dtype", DTYPES + [torch.float32])
@pytest.mark.parametrize("T,H,W", [(1, 8, 8), (3, 64, 72), (2, 40, 1280)])
def test_expansion(dvc, orc, dtype, T, H, W):
    f, f64 = dev(synthgen.frames(T, H, W), dtype)
    w, b = synthgen.expansion_weights()
    wd, w64 = dev(w, dtype)
    bd, b64 = dev(b, dtype)
    out = dvc.dvc_encode_pixelunshuffle(f, wd, bd)
    ref = orc.encode(f64, w64, b64, 8, MODE[dtype])
    err = rel_l2(host64(out), ref)
    assert err <= TOL[dtype], err


@pytest.mark.parametrize("c_lat", [64, 128, 192, 240, 256])
def test_expansion_latent_widths(dvc, orc, c_lat):
    # the encoder's staged epilogue: 64-column chunks (1..4 per tile, staging tiles cycled across tiles) when
    # c_lat % 64 == 0, 32/16-column chunks otherwise (240); 320 tiles on 148 CTAs: 2-3 tiles per CTA
    T = 16
    f, f64 = dev(synthgen.frames(T, 128, 1280), torch.bfloat16)
    w, b = synthgen.expansion_weights(c_lat=c_lat)
    wd, w64 = dev(w, torch.bfloat16)
    bd, b64 = dev(b, torch.bfloat16)
    out = host64(dvc.dvc_encode_pixelunshuffle(f, wd, bd))
    ref = orc.encode(f64, w64, b64, 8, "bf16")
    for t in range(T):   # per frame: a misplaced staging tile shows up as a frame-local error
        assert rel_l2(out[t], ref[t]) <= 1e-2


def test_expansion_identity_weights_exact(dvc, orc):   # P3 on the GPU: first 192 channels = unshuffle
    f, f64 = dev(synthgen.frames(2, 16, 24), torch.bfloat16)
    w = np.concatenate([np.eye(192), np.zeros((64, 192))]).astype(np.float32)
    out = dvc.dvc_encode_pixelunshuffle(f, dev(w, torch.bfloat16)[0], torch.zeros(256, dtype=torch.bfloat16,
                                                                                     device="cuda"))
    o = host64(out)
    assert np.array_equal(o[..., :192], orc.unshuffle(f64, 8)) and not o[..., 192:].any()


def test_expansion_720p_gop_sampled(dvc, orc):   # C2 at full size; frames 0 and 31 against the oracle
    f, f64 = dev(synthgen.frames(32, 720, 1280), torch.bfloat16)
    w, b = synthgen.expansion_weights()
    wd, w64 = dev(w, torch.bfloat16)
    bd, b64 = dev(b, torch.bfloat16)
    out = host64(dvc.dvc_encode_pixelunshuffle(f, wd, bd))
    for t in (0, 31):
        ref = orc.encode(f64[t:t + 1], w64, b64, 8, "bf16")
        assert rel_l2(out[t:t + 1], ref) <= 1e-2


# ---------------------------------------------------------------- a3 shift (bit-exact, same addressing as the producer)
@pytest.mark.parametrize("C,P", [(64, 8), (240, 8), (480, 8), (720, 8), (960, 8), (1440, 8), (1920, 8),
                                 (64, 2), (64, 4), (48, 8)])
def test_shift_gather_bitexact(dvc, orc, C, P):
    for T in (1, 2, 5, 12):
        x, x64 = dev(synthgen.normal((T, 3, 5, C), seed=T), torch.bfloat16)
        k, k64 = dev(synthgen.normal((3, 5, C // P), seed=99), torch.bfloat16)
        for carry, c64 in ((None, None), (k, k64)):
            out = dvc.dvc_debug_shift_gather(x, shift_p=P, carry_in=carry)
            ref, _ = orc.shift_batch(x64, c64, P)
            assert np.array_equal(host64(out), ref), (T, C, P)


def test_shift_gather_concat_sources(dvc, orc):
    x, x64 = dev(synthgen.normal((4, 3, 4, 480), seed=1), torch.float16)
    s, s64 = dev(synthgen.normal((4, 3, 4, 240), seed=2), torch.float16)
    out = dvc.dvc_debug_shift_gather(x, s, shift_p=8)
    ref, _ = orc.shift_batch(np.concatenate([x64, s64], -1), None, 8)
    assert np.array_equal(host64(out), ref)


# ---------------------------------------------------------------- a3-a8 ResBlock
def _run_block(dvc, w, x, xb=None, carry=None, carry_out=None, G=8, P=8):
    cb = 0 if xb is None else xb.shape[-1]
    p = dvc.ResBlockParams(w, x.shape[-1], cb, G, P)
    return dvc.dvc_resblock_tsm_forward(p, x, xb, carry_in=carry, carry_out=carry_out)


@pytest.mark.parametrize("with_carry", [False, True])
def test_resblock_fp32_config1(dvc, orc, with_carry):   # C1: T=8, 64 ch, 32x32, G=32, P=8, fp32, <= 1e-5
    w = synthgen.resblock_weights(64, 64)
    wd, w64 = rb_device(w, torch.float32)
    x, x64 = dev(synthgen.normal((8, 32, 32, 64)), torch.float32)
    k, k64 = dev(synthgen.normal((32, 32, 8), seed=7), torch.float32) if with_carry else (None, None)
    ko = torch.empty((32, 32, 8), device="cuda")
    out = _run_block(dvc, wd, x, carry=k, carry_out=ko, G=32)
    ref, kref = orc.resblock(x64, k64, w64, 32, 8)
    err = rel_l2(host64(out), ref)
    assert err <= 1e-5, err
    assert np.array_equal(host64(ko), kref)


@pytest.mark.parametrize("dtype", [torch.float32] + DTYPES)
@pytest.mark.parametrize("with_carry", [False, True])
@pytest.mark.parametrize("cin,cout,cb,T,H,W", [(32, 32, 0, 3, 9, 17), (48, 32, 0, 2, 16, 16), (64, 32, 32, 2, 7, 11),
                                                 (240, 240, 0, 2, 10, 13), (720, 240, 240, 1, 6, 9),
                                                 (1920, 960, 960, 2, 3, 5), (240, 480, 0, 1, 12, 20),
                                                 # H >= 32: the fused GN/SiLU/shift conv engine (8x16 halo boxes)
                                                 (240, 240, 0, 3, 40, 24), (720, 240, 240, 2, 34, 20),
                                                 (64, 32, 32, 2, 33, 9), (480, 480, 0, 2, 45, 16),
                                                 # > 74 CTA-pair tiles: slots cycle through raw and transformed chunks
                                                 (96, 32, 32, 6, 64, 72)])
def test_resblock_parity(dvc, orc, dtype, with_carry, cin, cout, cb, T, H, W):
    G = 8 if cin < 240 else 24
    w = synthgen.resblock_weights(cin, cout, seed=cin + cout)
    wd, w64 = rb_device(w, dtype)
    xa, xa64 = dev(synthgen.normal((T, H, W, cin - cb), seed=3), dtype)
    xb, xb64 = (dev(synthgen.normal((T, H, W, cb), seed=4), dtype) if cb else (None, None))
    k, k64 = dev(synthgen.normal((H, W, cin // 8), seed=5), dtype) if with_carry else (None, None)
    ko = torch.empty((H, W, cin // 8), dtype=dtype, device="cuda")
    out = _run_block(dvc, wd, xa, xb, carry=k, carry_out=ko, G=G)
    x64 = xa64 if xb is None else np.concatenate([xa64, xb64], -1)
    ref, kref = orc.resblock(x64, k64, w64, G, 8, mode=MODE[dtype])
    gate(host64(out), ref, dtype)
    assert np.array_equal(host64(ko), kref)          # G5: carry bytes, bit-exact


# P8 through the production engines (bit-exact): the residual branch of frame t depends on frame t-1's
# slice channels [0, C_in/P) (or the carry for t = 0) and on frame t's other channels, nothing else.
# A 1x1 shortcut with zero weights makes Out the residual branch exactly (0 + Y2).  C_in/P = 90 and 30
# straddle 8-channel vectors (the fused engine's per-vector TMA source selection) and 16-channel UMMA
# K steps; H >= 32 runs the fused GN/SiLU/shift engine, H < 32 the gn_silu gather + TMA engine.
@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("cin,cout,cb,T,H,W", [(720, 240, 240, 4, 34, 20), (240, 480, 0, 4, 40, 24),
                                                 (720, 240, 240, 4, 12, 20), (240, 480, 0, 4, 10, 13)])
def test_shift_isolation_through_the_engines(dvc, dtype, cin, cout, cb, T, H, W):
    G, P = 24, 8
    cs = cin // P
    w = synthgen.resblock_weights(cin, cout, seed=31)
    w["sc_w"][:] = 0
    w["sc_b"][:] = 0
    rng = np.random.default_rng(32)
    x = synthgen.normal((T, H, W, cin), seed=33)
    carry = synthgen.normal((H, W, cs), seed=34)

    def run(wts, xx, kk):
        wd, _ = rb_device(wts, dtype)
        xa = torch.from_numpy(np.ascontiguousarray(xx[..., :cin - cb])).to(dtype).cuda()
        xb = torch.from_numpy(np.ascontiguousarray(xx[..., cin - cb:])).to(dtype).cuda() if cb else None
        kd = None if kk is None else torch.from_numpy(kk).to(dtype).cuda()
        return _run_block(dvc, wd, xa, xb, carry=kd, G=G, P=P)

    noise = rng.standard_normal((H, W, cin)).astype(np.float32)
    for kk in (None, carry):
        base = run(w, x, kk)
        x_s = x.copy()
        x_s[1, ..., :cs] += noise[..., :cs]              # frame 1's slice: only frame 2 may move
        o = run(w, x_s, kk)
        assert torch.equal(o[[0, 1, 3]], base[[0, 1, 3]]) and not torch.equal(o[2], base[2])
        x_r = x.copy()
        x_r[1, ..., cs:] += noise[..., cs:]              # frame 1's other channels: only frame 1 may move
        o = run(w, x_r, kk)
        assert torch.equal(o[[0, 2, 3]], base[[0, 2, 3]]) and not torch.equal(o[1], base[1])
    # the carry reaches frame 0 only
    assert torch.equal(run(w, x, carry)[1:], run(w, x, None)[1:])
    # conv1's slice columns zero: nothing depends on frame t-1 or on the carry
    w0 = dict(w)
    w0["conv1_w"] = w["conv1_w"].copy()
    w0["conv1_w"][..., :cs] = 0
    base = run(w0, x, None)
    x_s = x.copy()
    x_s[:, ..., :cs] += rng.standard_normal((T, H, W, cs)).astype(np.float32)
    x_s[..., cs:] = x[..., cs:]
    assert torch.equal(run(w0, x, carry), base)
    # (changing every frame's slice changes nothing but the slice groups' own GN statistics, which only
    # scale zero-weight columns)
    assert torch.equal(run(w0, x_s, carry), base)
    # only the slice columns live: frame t's branch is a function of frame t-1's slice alone
    w1 = dict(w)
    w1["conv1_w"] = np.zeros_like(w["conv1_w"])
    w1["conv1_w"][..., :cs] = w["conv1_w"][..., :cs]
    base = run(w1, x, carry)
    x_r = x.copy()
    x_r[..., cs:] += rng.standard_normal((T, H, W, cin - cs)).astype(np.float32)
    assert torch.equal(run(w1, x_r, carry), base)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("H,W", [(8, 8), (36, 16)])
def test_resblock_identity_when_conv2_zero(dvc, dtype, H, W):   # P7 on the GPU, bit-exact
    w = synthgen.resblock_weights(64, 64)
    w["conv2_w"][:] = 0
    w["conv2_b"][:] = 0
    wd, _ = rb_device(w, dtype)
    x, _ = dev(synthgen.normal((3, H, W, 64)), dtype)
    out = _run_block(dvc, wd, x)
    assert torch.equal(out, x)


def test_resblock_legacy_gn_path(dvc, orc):   # G % P != 0: slice not whole groups -> per-element shifted GN pass
    dtype = torch.bfloat16
    w = synthgen.resblock_weights(240, 240, seed=11)
    wd, w64 = rb_device(w, dtype)
    x, x64 = dev(synthgen.normal((3, 40, 16, 240), seed=12), dtype)
    out = _run_block(dvc, wd, x, G=30)
    ref, _ = orc.resblock(x64, None, w64, 30, 8, mode="bf16")
    assert rel_l2(host64(out), ref) <= 1e-2


@pytest.mark.parametrize("dtype", DTYPES + [torch.float32])
@pytest.mark.parametrize("H,W", [(10, 12), (40, 17)])
def test_resblock_batch_equals_online_and_deterministic(dvc, dtype, H, W):   # P9 / G10 / G12, bit-exact
    w = synthgen.resblock_weights(240, 240)
    wd, _ = rb_device(w, dtype)
    T = 6
    x, _ = dev(synthgen.normal((T, H, W, 240)), dtype)
    full = _run_block(dvc, wd, x, G=24)
    again = _run_block(dvc, wd, x, G=24)
    assert torch.equal(full, again)
    carry, parts = None, []
    for t in range(T):
        ko = torch.empty((H, W, 30), dtype=dtype, device="cuda")
        parts.append(_run_block(dvc, wd, x[t:t + 1].contiguous(), carry=carry, carry_out=ko, G=24))
        carry = ko
    assert torch.equal(torch.cat(parts), full)


def test_resblock_720p_down0_sampled(dvc, orc):   # C3 shape (90x160, 240 ch, T=16, bf16); sampled frames
    dtype = torch.bfloat16
    T = 16
    w = synthgen.resblock_weights(240, 240)
    wd, w64 = rb_device(w, dtype)
    x, x64 = dev(synthgen.normal((T, 90, 160, 240)), dtype)
    out = host64(_run_block(dvc, wd, x, G=24))
    for t in (0, 9):
        lo = max(0, t - 1)
        carry = x64[lo - 1, ..., :30] if lo >= 1 else None
        ref, _ = orc.resblock(x64[lo:t + 1], carry, w64, 24, 8, mode="bf16")
        assert rel_l2(out[t], ref[-1]) <= 1e-2


def test_resblock_errors(dvc):
    w = synthgen.resblock_weights(64, 64)
    wd, _ = rb_device(w, torch.bfloat16)
    x = torch.zeros((2, 4, 4, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(dvc.DvcError) as e:
        _run_block(dvc, wd, x, G=7)
    assert e.value.name == "DVC_ERR_DIVISIBILITY"
    with pytest.raises(dvc.DvcError) as e:
        _run_block(dvc, wd, x, P=3)
    assert e.value.name == "DVC_ERR_DIVISIBILITY"
