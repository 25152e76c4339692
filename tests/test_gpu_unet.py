"""GPU parity of dvc_unet_decode_gop (a9, a10) against the oracle skeleton,
plus the bit-exact properties of the Batch-dimension OTSM across batching and
chunking."""
import numpy as np
import pytest
import torch

import synthgen
from tests.gpu_helpers import MODE, REG_STACK, TOL, dev, gate, host64, rel_l2

pytestmark = pytest.mark.gpu

SMALL = (32, 64, 96, 96)


@pytest.fixture(scope="module")
def dvc():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2601_20564_b200 as m
    m.device_check(0)
    return m


def _net(dvc, dtype, width, c_lat, h, w, max_T, G, seed=0, P=8):
    named = synthgen.unet_weights(width, c_lat, c_lat, seed=seed)
    cfg = dvc.unet_config(width, c_lat, c_lat, G, P, 1e-5, dtype, h, w, max_T)
    assert dvc.unet_weight_count(cfg) == sum(a.size for _, a in named)
    blob = dvc.pack_weights(named, dtype)
    exact = [(n, torch.from_numpy(a).to(dtype).double().numpy()) for n, a in named]
    return dvc.UNet(cfg, blob), exact


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16])
@pytest.mark.parametrize("h,w,T", [(12, 20, 3), (9, 14, 2), (64, 40, 2)])
def test_skeleton_small_parity(dvc, orc, dtype, h, w, T):
    net, wts = _net(dvc, dtype, SMALL, 32, h, w, 4, 8)
    lat, lat64 = dev(synthgen.normal((T, h, w, 32), 1), dtype)
    ctx, ctx64 = dev(synthgen.normal((T, h, w, 32), 5), dtype)
    co = torch.empty(net.carry_elems, dtype=dtype, device="cuda")
    out = dvc.dvc_unet_decode_gop(net, lat, ctx, carry_out=co)
    ref, kref = orc.skeleton(lat64, ctx64, wts, SMALL, G=8, P=8, mode=MODE[dtype])
    gate(host64(out), ref, dtype, reg=REG_STACK, ulps=32)
    # the carries are the GPU's own block inputs (computed activations): same tolerance
    packed = np.concatenate([k.ravel() for k in kref])
    assert rel_l2(host64(co), packed) <= TOL[dtype]


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("h,w", [(12, 20), (66, 36)])
def test_skeleton_batch_equals_online_and_chunks(dvc, dtype, h, w):   # G10, G11 (loopback), G12: bit-exact
    T = 6
    net, _ = _net(dvc, dtype, SMALL, 32, h, w, T, 8)
    lat, _ = dev(synthgen.normal((T, h, w, 32), 1), dtype)
    ctx, _ = dev(synthgen.normal((T, h, w, 32), 5), dtype)
    full = dvc.dvc_unet_decode_gop(net, lat, ctx)
    assert torch.equal(full, dvc.dvc_unet_decode_gop(net, lat, ctx))
    for chunks in ([1] * T, [2, 3, 1], [4, 2]):   # online (N=1) and ragged regroupings
        carry, parts, t0 = None, [], 0
        for n in chunks:
            ko = torch.empty(net.carry_elems, dtype=dtype, device="cuda")
            parts.append(dvc.dvc_unet_decode_gop(net, lat[t0:t0 + n].contiguous(), ctx[t0:t0 + n].contiguous(),
                                                 carry_in=carry, carry_out=ko))
            carry, t0 = ko, t0 + n
        assert torch.equal(torch.cat(parts), full), chunks


# f4: the shift ratio P (Fig. 8a sweep).  P = 2, 4 keep the slice whole GroupNorm groups (fused
# path); P = 16 does not (C_in/16 is not a multiple of C/G): the per-element shifted-statistics path.
@pytest.mark.parametrize("P", [2, 4, 16])
@pytest.mark.parametrize("h,w,T", [(12, 20, 3), (64, 40, 2)])
def test_skeleton_shift_ratio_sweep(dvc, orc, P, h, w, T):
    dtype = torch.bfloat16
    net, wts = _net(dvc, dtype, SMALL, 32, h, w, 4, 8, P=P)
    lat, lat64 = dev(synthgen.normal((T, h, w, 32), 1), dtype)
    ctx, ctx64 = dev(synthgen.normal((T, h, w, 32), 5), dtype)
    co = torch.empty(net.carry_elems, dtype=dtype, device="cuda")
    out = dvc.dvc_unet_decode_gop(net, lat, ctx, carry_out=co)
    ref, kref = orc.skeleton(lat64, ctx64, wts, SMALL, G=8, P=P, mode=MODE[dtype])
    assert rel_l2(host64(out), ref) <= TOL[dtype]
    # batch == online, bit-exact, at this P
    parts, carry = [], None
    for t in range(T):
        ko = torch.empty(net.carry_elems, dtype=dtype, device="cuda")
        parts.append(dvc.dvc_unet_decode_gop(net, lat[t:t + 1].contiguous(), ctx[t:t + 1].contiguous(),
                                             carry_in=carry, carry_out=ko))
        carry = ko
    assert torch.equal(torch.cat(parts), out)
    assert torch.equal(carry, co)


@pytest.mark.parametrize("h,w", [(12, 20), (66, 36)])
def test_streaming_decoder_graphs_bit_exact(dvc, h, w):   # f4: CUDA-graph online decode == batch decode
    dtype = torch.bfloat16
    T = 5
    net, _ = _net(dvc, dtype, SMALL, 32, h, w, T, 8)
    lat, _ = dev(synthgen.normal((T, h, w, 32), 1), dtype)
    ctx, _ = dev(synthgen.normal((T, h, w, 32), 5), dtype)
    full = dvc.dvc_unet_decode_gop(net, lat, ctx)
    sd = dvc.StreamingDecoder(net)
    for _ in range(2):   # a reset starts a new chain: the same outputs again
        sd.reset()
        outs = [sd.step(lat[t], ctx[t]).clone() for t in range(T)]
        assert torch.equal(torch.cat(outs), full)


def test_skeleton_real_widths_small_latent(dvc, orc):   # R1 widths 240/480/960 at a 16x24 latent, bf16
    dtype = torch.bfloat16
    h, w, T = 16, 24, 2
    net, wts = _net(dvc, dtype, (240, 480, 960, 960), 256, h, w, T, 24)
    lat, lat64 = dev(synthgen.normal((T, h, w, 256), 1), dtype)
    ctx, ctx64 = dev(synthgen.normal((T, h, w, 256), 5), dtype)
    out = dvc.dvc_unet_decode_gop(net, lat, ctx)
    ref, _ = orc.skeleton(lat64, ctx64, wts, G=24, P=8, mode="bf16")
    assert rel_l2(host64(out), ref) <= 1e-2


@pytest.mark.slow
def test_skeleton_720p_frame0(dvc, orc):   # C3 workload (720p, T=16, bf16); frame 0 depends on frame 0 only
    dtype = torch.bfloat16
    h, w, T = 90, 160, 16
    net, wts = _net(dvc, dtype, (240, 480, 960, 960), 256, h, w, T, 24)
    lat, lat64 = dev(synthgen.normal((T, h, w, 256), 1), dtype)
    ctx, ctx64 = dev(synthgen.normal((T, h, w, 256), 5), dtype)
    out = host64(dvc.dvc_unet_decode_gop(net, lat, ctx))
    assert np.isfinite(out).all()
    ref, _ = orc.skeleton(lat64[:1], ctx64[:1], wts, G=24, P=8, mode="bf16")
    assert rel_l2(out[:1], ref) <= 1e-2
