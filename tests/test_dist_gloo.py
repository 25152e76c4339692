"""Multi-process (gloo, world size 2, CPU) test of the multi-GPU protocol:
contiguous frame chunks per rank, and before every ResBlock k rank r sends the
C_in/P slice of its last frame's block input to rank r+1 and receives rank r-1's
as its carry (the inter-batch shift of P:151 across ranks).  Run on the fp64
oracle: the sharded result must equal the unsharded skeleton exactly."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthgen

SMALL = (32, 64, 96, 96)


def chunk(T, world, rank):
    """Contiguous chunks; the remainder goes to the last ranks (R18)."""
    base, rem = divmod(T, world)
    sizes = [base + (1 if r >= world - rem else 0) for r in range(world)]
    t0 = sum(sizes[:rank])
    return t0, t0 + sizes[rank]


def _worker(rank, world, port, T, out_q):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h, w = 6, 10
    wts = [(n, a.astype(np.float64)) for n, a in synthgen.unet_weights(SMALL, 32, 32)]
    lat, ctx = synthgen.normal((T, h, w, 32), 1), synthgen.normal((T, h, w, 32), 5)
    a, b = chunk(T, world, rank)

    def halo(k, X):
        c = X.shape[-1] // 8
        req = None
        if rank < world - 1:
            req = dist.isend(torch.from_numpy(np.ascontiguousarray(X[-1, ..., :c])), rank + 1, tag=k)
        carry = None
        if rank > 0:
            buf = torch.empty(X.shape[1:-1] + (c,), dtype=torch.float64)
            dist.recv(buf, rank - 1, tag=k)
            carry = buf.numpy()
        if req is not None:
            req.wait()
        return carry

    out, _ = oracle.skeleton(lat[a:b], ctx[a:b], wts, SMALL, G=8, P=8, halo=halo)
    out_q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("T,world", [(4, 2), (5, 2)])
def test_sharded_halo_equals_unsharded(orc, T, world):
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = 29500 + T * 7 + world
    procs = [ctx_mp.Process(target=_worker, args=(r, world, port, T, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    sharded = np.concatenate([res[r] for r in range(world)])
    h, w = 6, 10
    wts = [(n, a.astype(np.float64)) for n, a in synthgen.unet_weights(SMALL, 32, 32)]
    lat, ctx = synthgen.normal((T, h, w, 32), 1), synthgen.normal((T, h, w, 32), 5)
    ref, _ = orc.skeleton(lat, ctx, wts, SMALL, G=8, P=8)
    assert np.array_equal(sharded, ref)


def test_chunking_covers_and_is_contiguous():
    for T in range(1, 40):
        for world in (1, 2, 3, 4, 8):
            spans = [chunk(T, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == T
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
