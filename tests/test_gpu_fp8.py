"""GPU checks of the f4 fp8 variant: E4M3 quantisation bit-exact against the oracle's rounding
(R32), and the fp8 tcgen05 convolution (kind::f8f6f4 on the TMA engine) against the exact
dequantised convolution."""
import numpy as np
import pytest
import torch

import synthgen
from tests.gpu_helpers import host64, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dvc():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2601_20564_b200 as m
    m.device_check(0)
    return m


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32])
@pytest.mark.parametrize("scale", [1.0, 0.013, 0.25])
def test_quantize_e4m3_bit_exact(dvc, orc, dtype, scale):
    x = torch.from_numpy(synthgen.normal((4096,), 31, scale=3.0)).to(dtype)
    x[:4] = torch.tensor([1e5, -1e5, 0.0, 448.0 * scale])
    q = dvc.dvc_quantize_e4m3(x.cuda(), scale).cpu()
    got = q.view(torch.float8_e4m3fn).float().double().numpy()
    ref = orc.quantize_e4m3(x.float().numpy(), scale)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("out_dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("T,H,W,cin,cout,k", [(2, 12, 20, 64, 64, 3), (1, 45, 80, 480, 480, 3), (2, 9, 14, 96, 48, 1),
                                               (1, 23, 40, 960, 960, 3)])
def test_conv_fp8_parity(dvc, orc, out_dtype, T, H, W, cin, cout, k):
    x = torch.from_numpy(synthgen.normal((T, H, W, cin), 32)).cuda()
    w = torch.from_numpy(synthgen.normal((cout, k, k, cin), 33, scale=1.0 / np.sqrt(k * k * cin))).cuda()
    b = torch.from_numpy(synthgen.normal((cout,), 34, scale=0.1)).to(out_dtype)
    sx = float(x.abs().max()) / 448.0
    sw = float(w.abs().max()) / 448.0
    x8, w8 = dvc.dvc_quantize_e4m3(x, sx), dvc.dvc_quantize_e4m3(w, sw)
    y = dvc.dvc_conv_fp8(x8, sx, w8, sw, b.cuda(), out_dtype=out_dtype)
    qx = x8.cpu().view(torch.float8_e4m3fn).double().numpy()
    qw = w8.cpu().view(torch.float8_e4m3fn).double().numpy()
    ref = orc.conv_fp8(qx, sx, qw, sw, b.double().numpy())
    assert rel_l2(host64(y), ref) <= 1e-2                          # accumulation order + 16-bit output
    exact = orc.conv2d(x.cpu().double().numpy(), w.cpu().double().numpy(), b.double().numpy(), 1, k // 2)
    assert rel_l2(host64(y), exact) <= 8e-2                        # E4M3 quantisation error (3 mantissa bits)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_dvc_conv_parity(dvc, orc, dtype):
    x = torch.from_numpy(synthgen.normal((2, 12, 20, 64), 35)).to(dtype)
    w = torch.from_numpy(synthgen.normal((48, 3, 3, 64), 36, scale=1 / 24)).to(dtype)
    b = torch.from_numpy(synthgen.normal((48,), 37, scale=0.1)).to(dtype)
    y = dvc.dvc_conv(x.cuda(), w.cuda(), b.cuda())
    ref = orc.conv2d(x.double().numpy(), w.double().numpy(), b.double().numpy())
    assert rel_l2(host64(y), ref) <= (1e-2 if dtype != torch.float32 else 1e-5)


@pytest.mark.parametrize("H,W,cin,cout", [(12, 20, 960, 960), (23, 40, 480, 960)])
def test_narrow_n_tiles_are_bit_exact(dvc, H, W, cin, cout):
    # T-adaptive N tiles (the TMA engine narrows its N tile while a call fills less than half a wave):
    # T = 1 runs narrow tiles, T = 48 the full-width ones; N-splitting keeps every output's K order, so
    # the frames must agree bit for bit
    T = 48
    x = torch.from_numpy(synthgen.normal((T, H, W, cin), 41)).to(torch.bfloat16).cuda()
    w = torch.from_numpy(synthgen.normal((cout, 3, 3, cin), 42, scale=1 / 90)).to(torch.bfloat16).cuda()
    b = torch.from_numpy(synthgen.normal((cout,), 43, scale=0.1)).to(torch.bfloat16).cuda()
    full = dvc.dvc_conv(x, w, b)
    for t in (0, 17, T - 1):
        one = dvc.dvc_conv(x[t:t + 1].contiguous(), w, b)
        assert torch.equal(one[0], full[t]), t


def test_odd_epilogue_chunk_count_is_repeatable(dvc, orc):
    # 1x1 conv 128 -> 64 on the TMA engine: two epilogue warpgroups, ONE 32-column staged chunk each per
    # work item (an odd count), ~20 items per CTA pair. The staging-buffer parity runs across items, so
    # no item writes the buffer whose TMA store from the previous item may still be reading it: every
    # run, and every frame run alone, must give the same bits
    T, H, W, cin, cout = 16, 90, 160, 128, 64
    x = torch.from_numpy(synthgen.normal((T, H, W, cin), 51)).to(torch.bfloat16).cuda()
    w = torch.from_numpy(synthgen.normal((cout, 1, 1, cin), 52, scale=1 / 12)).to(torch.bfloat16).cuda()
    b = torch.from_numpy(synthgen.normal((cout,), 53, scale=0.1)).to(torch.bfloat16).cuda()
    ref = dvc.dvc_conv(x, w, b)
    for _ in range(20):
        assert torch.equal(dvc.dvc_conv(x, w, b), ref)
    one = dvc.dvc_conv(x[5:6].contiguous(), w, b)
    assert torch.equal(one[0], ref[5])
    # values: a corner crop against the fp64 oracle (a 1x1 conv is per pixel)
    xc = x[:1, :8, :16].cpu().double().numpy()
    exact = orc.conv2d(xc, w.cpu().double().numpy(), b.cpu().double().numpy())
    assert rel_l2(host64(ref[:1, :8, :16]), exact) <= 1e-2
