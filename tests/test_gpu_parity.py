"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle.

Bit-exact for index work (unshuffle, shift, carry); rel-L2 <= 1e-2 for
16-bit outputs against the storage-rounding-emulated oracle (R15/R16) and
<= 1e-5 for the fp32 validation mode against the pure fp64 oracle.
"""
import numpy as np
import pytest
import torch

import synthgen
from tests.gpu_helpers import MODE, TOL, dev, host64, rb_device, rel_l2

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
@pytest.mark.parametrize("cin,cout,cb,T,H,W", [(32, 32, 0, 3, 9, 17), (48, 32, 0, 2, 16, 16), (64, 32, 32, 2, 7, 11),
                                                 (240, 240, 0, 2, 10, 13), (720, 240, 240, 1, 6, 9),
                                                 (1920, 960, 960, 2, 3, 5), (240, 480, 0, 1, 12, 20),
                                                 # H >= 32: the fused GN/SiLU/shift conv engine (8x16 halo boxes)
                                                 (240, 240, 0, 3, 40, 24), (720, 240, 240, 2, 34, 20),
                                                 (64, 32, 32, 2, 33, 9), (480, 480, 0, 2, 45, 16),
                                                 # > 74 CTA-pair tiles: slots cycle through raw and transformed chunks
                                                 (96, 32, 32, 6, 64, 72)])
def test_resblock_parity(dvc, orc, dtype, cin, cout, cb, T, H, W):
    G = 8 if cin < 240 else 24
    w = synthgen.resblock_weights(cin, cout, seed=cin + cout)
    wd, w64 = rb_device(w, dtype)
    xa, xa64 = dev(synthgen.normal((T, H, W, cin - cb), seed=3), dtype)
    xb, xb64 = (dev(synthgen.normal((T, H, W, cb), seed=4), dtype) if cb else (None, None))
    k, k64 = dev(synthgen.normal((H, W, cin // 8), seed=5), dtype)
    ko = torch.empty((H, W, cin // 8), dtype=dtype, device="cuda")
    out = _run_block(dvc, wd, xa, xb, carry=k, carry_out=ko, G=G)
    x64 = xa64 if xb is None else np.concatenate([xa64, xb64], -1)
    ref, kref = orc.resblock(x64, k64, w64, G, 8, mode=MODE[dtype])
    err = rel_l2(host64(out), ref)
    assert err <= TOL[dtype], err
    assert np.array_equal(host64(ko), kref)          # G5: carry bytes, bit-exact


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
