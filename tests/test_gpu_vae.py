"""GPU parity of f2, the pruned VAE decoder (dvc_vae_decode), against the fp64 oracle
(oracle.vae_decode, readings R29-R31), plus the single-head head_dim-256 attention it uses and
the shift-free ResBlock (shift_p = 0)."""
import numpy as np
import pytest
import torch

import synthgen
from tests.gpu_helpers import MODE, TOL, dev, host64, rb_device, rel_l2

pytestmark = pytest.mark.gpu

VSMALL = (16, 32, 48, 48)


@pytest.fixture(scope="module")
def dvc():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2601_20564_b200 as m
    m.device_check(0)
    return m


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32])
@pytest.mark.parametrize("T,N", [(2, 300), (1, 129)])
def test_attention_head_dim_256(dvc, orc, dtype, T, N):
    C = 256
    qkv, q64 = dev(synthgen.normal((T, N, 3 * C), 21, scale=0.5), dtype)
    out = dvc.dvc_attention_forward(qkv, 256)
    ref = orc.rnd(orc.attention(q64[..., :C], q64[..., C:2 * C], q64[..., 2 * C:], 256), MODE[dtype])
    assert rel_l2(host64(out), ref) <= TOL[dtype]


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("cin,cout,H,W", [(48, 48, 12, 20), (64, 32, 40, 48)])
def test_resblock_without_shift(dvc, orc, dtype, cin, cout, H, W):
    T = 2
    w = synthgen.resblock_weights(cin, cout)
    wd, wh = rb_device(w, dtype)
    p = dvc.ResBlockParams(wd, cin, 0, 8, 0)          # shift_p = 0: no temporal shift
    x, x64 = dev(synthgen.normal((T, H, W, cin), 3), dtype)
    y = dvc.dvc_resblock_tsm_forward(p, x)
    ref = orc.vae_resblock(x64, wh, 8, 1e-5, MODE[dtype])
    assert rel_l2(host64(y), ref) <= TOL[dtype]


def _vae(dvc, dtype, h, w, T, mid_attn=True, attn_scale=2.0):
    named = synthgen.vae_weights(VSMALL, 32, mid_attn=mid_attn, attn_scale=attn_scale)
    v = dvc.VAE(dvc.pack_weights(named, dtype), VSMALL, 32, 3, 8, 1e-6, mid_attn, dtype, h, w, T)
    assert v.weight_count() == sum(a.size for _, a in named)
    exact = [(n, torch.from_numpy(a).to(dtype).double().numpy()) for n, a in named]
    return v, exact


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32])
@pytest.mark.parametrize("h,w,T,mid", [(3, 4, 2, True), (6, 8, 2, True), (5, 7, 1, False),
                                        # H >= 32: the fused engine, whose conv2 epilogue writes the 2x
                                        # upsampled block output directly (folded nearest)
                                        (32, 8, 1, True)])
def test_vae_decoder_parity(dvc, orc, dtype, h, w, T, mid):
    v, wts = _vae(dvc, dtype, h, w, T, mid)
    lat, lat64 = dev(synthgen.normal((T, h, w, 32), 1), dtype)
    out = dvc.dvc_vae_decode(v, lat)
    assert out.shape == (T, 8 * h, 8 * w, 3)
    ref = orc.vae_decode(lat64, wts, VSMALL, G=8, eps=1e-6, mid_attn=mid, mode=MODE[dtype])
    err = rel_l2(host64(out), ref)
    tol = TOL[dtype]
    if dtype == torch.bfloat16:
        # R31: bf16 storage alone moves the decoder output by 1.4e-2..2.3e-2 (emulated oracle vs pure
        # fp64), above the 1e-2 ResBlock gate, so end to end bf16 is gated at twice that intrinsic
        # error; its ResBlocks are gated at 1e-2 one by one (test_resblock_without_shift)
        pure = orc.vae_decode(lat64, wts, VSMALL, G=8, eps=1e-6, mid_attn=mid, mode=None)
        tol = max(tol, 2 * rel_l2(ref, pure))
    assert err <= tol, (err, tol)
    assert torch.equal(out, dvc.dvc_vae_decode(v, lat))              # deterministic


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("h,w,T", [(4, 9, 2), (5, 4, 1)])
def test_vae_decoder_parity_real_widths(dvc, orc, dtype, h, w, T):
    # the paper's decoder widths (64, 128, 256, 256; 32 groups) at small latents: the 64-channel output
    # head (dvc_conv_out.cu, KS = 4) with ragged 32-pixel tiles (72 = 2 x 32 + 8) and a frame narrower
    # than one tile (32 pixels, 40 rows = 5 tiles), against the oracle end to end
    named = synthgen.vae_weights(seed=11)
    v = dvc.VAE(dvc.pack_weights(named, dtype), dtype=dtype, h=h, w=w, max_T=T)
    exact = [(n, torch.from_numpy(a).to(dtype).double().numpy()) for n, a in named]
    lat, lat64 = dev(synthgen.normal((T, h, w, 256), 4), dtype)
    out = dvc.dvc_vae_decode(v, lat)
    assert out.shape == (T, 8 * h, 8 * w, 3)
    ref = orc.vae_decode(lat64, exact, mode=MODE[dtype])
    err = rel_l2(host64(out), ref)
    tol = TOL[dtype]
    if dtype == torch.bfloat16:   # R31, as in test_vae_decoder_parity
        tol = max(tol, 2 * rel_l2(ref, orc.vae_decode(lat64, exact, mode=None)))
    assert err <= tol, (err, tol)


def test_vae_frames_independent(dvc):
    h, w = 6, 8
    v, _ = _vae(dvc, torch.bfloat16, h, w, 3)
    lat, _ = dev(synthgen.normal((3, h, w, 32), 1), torch.bfloat16)
    full = dvc.dvc_vae_decode(v, lat)
    for t in range(3):
        assert torch.equal(dvc.dvc_vae_decode(v, lat[t:t + 1].contiguous())[0], full[t])


def test_error_paths_return_before_launch(dvc):
    # unsupported shapes fail loudly with a status, never a silent fallback (include/dvc.h)
    qkv = torch.zeros((1, 10, 3 * 80), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(dvc.DvcError, match="UNSUPPORTED"):
        dvc.dvc_attention_forward(qkv, 40)                       # head_dim 40 not in {16,32,48,64,256}
    with pytest.raises(dvc.DvcError, match="DIVISIBILITY"):
        dvc.dvc_attention_forward(torch.zeros((1, 10, 3 * 96), dtype=torch.bfloat16, device="cuda"), 64)
    named = synthgen.vae_weights((16, 32, 48, 80), 32)
    with pytest.raises(dvc.DvcError, match="UNSUPPORTED"):       # single-head attention of width 80
        dvc.VAE(dvc.pack_weights(named, torch.bfloat16), (16, 32, 48, 80), 32, 3, 8, 1e-6, True, torch.bfloat16,
                4, 4, 1)
    x8 = torch.zeros((1, 4, 4, 48), dtype=torch.uint8, device="cuda")
    w8 = torch.zeros((16, 3, 3, 48), dtype=torch.uint8, device="cuda")
    with pytest.raises(dvc.DvcError, match="UNSUPPORTED"):       # fp8 conv needs C_in % 32
        dvc.dvc_conv_fp8(x8, 1.0, w8, 1.0)


@pytest.mark.slow
def test_vae_720p_frames_independent_and_deterministic(dvc):
    # the bench's real decoder at 720p (90x160 latent -> 720x1280): per-frame == batched, bit-exact
    v = dvc.VAE(dvc.pack_weights(synthgen.vae_weights(), torch.bfloat16), dtype=torch.bfloat16, h=90, w=160, max_T=2)
    lat, _ = dev(synthgen.normal((2, 90, 160, 256), 1), torch.bfloat16)
    full = dvc.dvc_vae_decode(v, lat)
    assert full.shape == (2, 720, 1280, 3) and torch.isfinite(full.float()).all()
    assert torch.equal(full, dvc.dvc_vae_decode(v, lat))
    assert torch.equal(dvc.dvc_vae_decode(v, lat[1:].contiguous())[0], full[1])



@pytest.mark.slow
def test_1080p_sizes_no_index_overflow(dvc):
    # 1080p latents (135x240): level-3 VAE tensors of 8 frames exceed 2^31 bytes; batched == per-frame /
    # chunked bit for bit for the VAE decoder and the full U-Net (32-bit index overflow would break it)
    dt, h, w = torch.bfloat16, 135, 240
    vae = dvc.VAE(dvc.pack_weights(synthgen.vae_weights(), dt), dtype=dt, h=h, w=w, max_T=8)
    lat, _ = dev(synthgen.normal((8, h, w, 256), 7), dt)
    fr = dvc.dvc_vae_decode(vae, lat)
    assert torch.isfinite(fr.float()).all()
    assert torch.equal(dvc.dvc_vae_decode(vae, lat[7:].contiguous())[0], fr[7])
    del fr
    W = (240, 480, 960, 960)
    net = dvc.UNet(dvc.unet_config(W, 256, 256, 24, 8, 1e-5, dt, h, w, 4, head_dim=48),
                   dvc.pack_weights(synthgen.unet_weights(W, attention=True), dt))
    ctx, _ = dev(synthgen.normal((4, h, w, 256), 5), dt)
    full = dvc.dvc_unet_decode_gop(net, lat[:4].contiguous(), ctx)
    co = torch.empty(net.carry_elems, dtype=dt, device="cuda")
    a = dvc.dvc_unet_decode_gop(net, lat[:3].contiguous(), ctx[:3].contiguous(), carry_out=co)
    b = dvc.dvc_unet_decode_gop(net, lat[3:4].contiguous(), ctx[3:].contiguous(), carry_in=co)
    assert torch.isfinite(full.float()).all() and torch.equal(torch.cat([a, b]), full)
