"""GPU checks of f3, the Asynchronous and Parallel Decoding Pipeline: frames pushed
one at a time from a producer stream and decoded N at a time on the pipeline's stream come out
bit-identical to one dvc_unet_decode_gop call over the whole chain (batch == online),
with N-1 frames of latency, ragged tails (R18) and chain resets (R9)."""
import pytest
import torch

import synthgen
from tests.gpu_helpers import dev

pytestmark = pytest.mark.gpu

SMALL = (32, 64, 96, 96)


@pytest.fixture(scope="module")
def dvc():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2601_20564_b200 as m
    m.device_check(0)
    return m


def _net(dvc, h, w, max_T, head_dim=0):
    named = synthgen.unet_weights(SMALL, 32, 32, attention=head_dim > 0)
    cfg = dvc.unet_config(SMALL, 32, 32, 8, 8, 1e-5, torch.bfloat16, h, w, max_T, head_dim=head_dim)
    return dvc.UNet(cfg, dvc.pack_weights(named, torch.bfloat16))


@pytest.mark.parametrize("N,K,T,head_dim", [(4, 2, 12, 0), (4, 3, 10, 0), (3, 1, 7, 16), (1, 2, 5, 0)])
def test_pipeline_equals_one_call(dvc, N, K, T, head_dim):
    h, w = 12, 20
    net = _net(dvc, h, w, max(N, T), head_dim)
    lat, _ = dev(synthgen.normal((T, h, w, 32), 1), torch.bfloat16)
    ctx, _ = dev(synthgen.normal((T, h, w, 32), 5), torch.bfloat16)
    ref = dvc.dvc_unet_decode_gop(net, lat, ctx)
    pipe = dvc.Pipeline(net, N, K)
    producer = torch.cuda.Stream()
    got, latency = {}, []
    for t in range(T):
        with torch.cuda.stream(producer):
            pipe.push(lat[t], ctx[t])
        while True:
            r = pipe.pop()
            if r is None:
                break
            first, x = r
            for i in range(x.shape[0]):
                got[first + i] = x[i].clone()
                latency.append(t - (first + i))
    pipe.flush()
    while (r := pipe.pop()) is not None:
        first, x = r
        for i in range(x.shape[0]):
            got[first + i] = x[i].clone()
            latency.append(T - 1 - (first + i))
    torch.cuda.synchronize()
    assert sorted(got) == list(range(T))
    out = torch.stack([got[t] for t in range(T)])
    assert torch.equal(out, ref)
    assert max(latency) <= N - 1
    if T >= N:
        assert max(latency) == N - 1                     # N-1 frame latency


def test_pipeline_reset_starts_new_chain(dvc):
    h, w, N = 12, 20, 2
    net = _net(dvc, h, w, 4)
    lat, _ = dev(synthgen.normal((6, h, w, 32), 1), torch.bfloat16)
    ctx, _ = dev(synthgen.normal((6, h, w, 32), 5), torch.bfloat16)
    ref_a = dvc.dvc_unet_decode_gop(net, lat[:3], ctx[:3])
    ref_b = dvc.dvc_unet_decode_gop(net, lat[3:], ctx[3:])
    pipe = dvc.Pipeline(net, N, 4)
    outs = []
    for t in range(6):
        if t == 3:
            pipe.reset()                                  # GOP boundary: zero carry (R8, R9)
        pipe.push(lat[t], ctx[t])
    pipe.flush()
    while (r := pipe.pop()) is not None:
        outs.append(r[1].clone())
    torch.cuda.synchronize()
    out = torch.cat(outs)
    assert torch.equal(out[:3], ref_a) and torch.equal(out[3:], ref_b)


def test_pipeline_full_fifo_is_an_error(dvc):
    net = _net(dvc, 12, 20, 2)
    lat, _ = dev(synthgen.normal((5, 12, 20, 32), 1), torch.bfloat16)
    pipe = dvc.Pipeline(net, 2, 2)
    for t in range(4):
        pipe.push(lat[t], lat[t])
    with pytest.raises(dvc.DvcError):
        pipe.push(lat[4], lat[4])
    assert pipe.pop() is not None
    pipe.push(lat[4], lat[4])


def test_pipeline_with_vae_decoder_outputs_frames(dvc):
    # the whole Frame Reconstructor in the pipeline: U-Net then the VAE decoder ("pass them
    # through the U-Net and VAE Decoder in parallel"); equal to the two calls made directly
    h, w, N, T = 8, 10, 2, 5
    net = _net(dvc, h, w, T)
    VS = (16, 32, 48, 48)
    vae = dvc.VAE(dvc.pack_weights(synthgen.vae_weights(VS, 32), torch.bfloat16), VS, 32, 3, 8, 1e-6, True,
                  torch.bfloat16, h, w, T)
    lat, _ = dev(synthgen.normal((T, h, w, 32), 1), torch.bfloat16)
    ctx, _ = dev(synthgen.normal((T, h, w, 32), 5), torch.bfloat16)
    ref = dvc.dvc_vae_decode(vae, dvc.dvc_unet_decode_gop(net, lat, ctx))
    pipe = dvc.Pipeline(net, N, 3, vae=vae)
    got = {}
    for t in range(T):
        pipe.push(lat[t], ctx[t])
        while (r := pipe.pop()) is not None:
            for i in range(r[1].shape[0]):
                got[r[0] + i] = r[1][i].clone()
    pipe.flush()
    while (r := pipe.pop()) is not None:
        for i in range(r[1].shape[0]):
            got[r[0] + i] = r[1][i].clone()
    torch.cuda.synchronize()
    out = torch.stack([got[t] for t in range(T)])
    assert out.shape == (T, 8 * h, 8 * w, 3)
    assert torch.equal(out, ref)



@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_pipeline_matches_oracle(dvc, orc, dtype):
    """f3 against the fp64 oracle (not only against the direct call): frames pushed one at a time,
    decoded N at a time with the inter-batch carry, popped in order == oracle.skeleton over the whole
    chain (storage-rounding emulation of dtype; R15/R16 gates per frame)."""
    from tests.gpu_helpers import MODE, REG_STACK, gate, host64
    h, w, N, T = 12, 20, 3, 7
    named = synthgen.unet_weights(SMALL, 32, 32, seed=3)
    cfg = dvc.unet_config(SMALL, 32, 32, 8, 8, 1e-5, dtype, h, w, N)
    net = dvc.UNet(cfg, dvc.pack_weights(named, dtype))
    lat, lat64 = dev(synthgen.normal((T, h, w, 32), 41), dtype)
    ctx, ctx64 = dev(synthgen.normal((T, h, w, 32), 42), dtype)
    pipe = dvc.Pipeline(net, N, 2)
    got = {}

    def drain():
        while (r := pipe.pop()) is not None:
            first, x = r
            for i in range(x.shape[0]):
                got[first + i] = x[i].clone()

    for t in range(T):
        pipe.push(lat[t], ctx[t])
        drain()
    pipe.flush()
    drain()
    torch.cuda.synchronize()
    out = torch.stack([got[t] for t in range(T)])
    exact = [(n, torch.from_numpy(a).to(dtype).double().numpy()) for n, a in named]
    ref, _ = orc.skeleton(lat64, ctx64, exact, SMALL, G=8, P=8, mode=MODE[dtype])
    gate(host64(out), ref, dtype, "pipeline", reg=REG_STACK, ulps=32)
