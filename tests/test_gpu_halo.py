"""GPU tests of the multi-GPU halo (row e; "passes the partial channels of
the last sample ... to the subsequent batch") on ONE GPU:

* loopback: `world` ranks of one process, each on its own CUDA stream, connected in-process
  (dvc_comm_connect_local), all enqueued without host synchronisation -- the P2P transport's copy-engine
  peer copies, stream-memory arrival flags, epoch slots and acknowledgements all run, and the
  concatenated chunks must equal the single-rank decode BIT FOR BIT (carry_out of the last rank too),
  over several consecutive calls (epochs >= 3 exercise the slot reuse / acknowledgement wait);
* IPC: two processes on cuda:0 connected with CUDA IPC handles gathered over torch.distributed (gloo)
  -- the cross-process path of the bench -- against the single-process decode, bit for bit.
"""
import os

import numpy as np
import pytest
import torch

import synthgen

pytestmark = pytest.mark.gpu

SMALL = (32, 64, 96, 96)


@pytest.fixture(scope="module")
def dvc():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2601_20564_b200 as m
    m.device_check(0)
    return m


def _net(dvc, dtype, width, c, h, w, max_T, G, attention=False, head_dim=0):
    named = synthgen.unet_weights(width, c, c, attention=attention)
    cfg = dvc.unet_config(width, c, c, G, 8, 1e-5, dtype, h, w, max_T, head_dim=head_dim)
    return dvc.UNet(cfg, dvc.pack_weights(named, dtype))


def _inputs(T, h, w, c, dtype, seed):
    lat = torch.from_numpy(synthgen.normal((T, h, w, c), seed)).to(dtype).cuda()
    ctx = torch.from_numpy(synthgen.normal((T, h, w, c), seed + 50)).to(dtype).cuda()
    return lat, ctx


def _loopback(dvc, net, comms, lat, ctx, carry_out):
    """One decode call per rank, each on its own stream, enqueued back to back (no host sync)."""
    world = len(comms)
    T = lat.shape[0]
    bounds = dvc.chunk_bounds(T, world)
    streams = [torch.cuda.Stream() for _ in range(world)]
    start = torch.cuda.Event()
    start.record()
    outs = []
    for r, (a, b) in enumerate(bounds):
        s = streams[r]
        s.wait_event(start)
        with torch.cuda.stream(s):
            ws = torch.empty(net.workspace_size(b - a), dtype=torch.uint8, device="cuda")
            out = torch.empty((b - a,) + tuple(lat.shape[1:3]) + (net.cfg.c_lat,), dtype=lat.dtype, device="cuda")
            dvc.dvc_unet_decode_gop(net, lat[a:b], ctx[a:b], comm=comms[r], out=out, workspace=ws,
                                    carry_out=carry_out if r == world - 1 else None, stream=s)
            outs.append(out)
    torch.cuda.synchronize()
    return torch.cat(outs)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("world,T,h,w", [(2, 6, 12, 20), (3, 7, 12, 20), (4, 8, 66, 36), (2, 5, 40, 64)])
def test_loopback_halo_equals_single_rank(dvc, dtype, world, T, h, w):
    net = _net(dvc, dtype, SMALL, 32, h, w, T, 8)
    comms = dvc.Comm.local_group(world, net)
    for call in range(4):        # 4 epochs: both slots used twice, acknowledgement waits from epoch 3
        lat, ctx = _inputs(T, h, w, 32, dtype, 10 + call)
        ref_k = torch.empty(net.carry_elems, dtype=dtype, device="cuda")
        ref = dvc.dvc_unet_decode_gop(net, lat, ctx, carry_out=ref_k)
        k = torch.full((net.carry_elems,), float("nan"), dtype=dtype, device="cuda")
        got = _loopback(dvc, net, comms, lat, ctx, k)
        assert torch.equal(got, ref), f"call {call}: sharded decode differs from world 1"
        assert torch.equal(k, ref_k), f"call {call}: carry_out of the last rank differs"
    for c in comms:
        c.close()


def test_loopback_halo_real_widths_full_unet(dvc):
    """The 720p channel widths (slices of 30..240 channels) with the Transformer2D blocks (the halo is
    released after the block's attention), world 4 at a reduced latent size."""
    dtype, T, h, w = torch.bfloat16, 8, 24, 40
    net = _net(dvc, dtype, (240, 480, 960, 960), 256, h, w, T, 24, attention=True, head_dim=48)
    comms = dvc.Comm.local_group(4, net)
    for call in range(3):
        lat, ctx = _inputs(T, h, w, 256, dtype, 20 + call)
        ref = dvc.dvc_unet_decode_gop(net, lat, ctx)
        assert torch.equal(_loopback(dvc, net, comms, lat, ctx, None), ref)


def test_halo_comm_argument_errors(dvc):
    lib = dvc.lib()
    net = _net(dvc, torch.bfloat16, SMALL, 32, 12, 20, 4, 8)
    c0, c1 = dvc.Comm(0, 2, net, _connect=False), dvc.Comm(1, 2, net, _connect=False)
    lat, ctx = _inputs(2, 12, 20, 32, torch.bfloat16, 1)
    with pytest.raises(dvc.DvcError):          # not connected: refused before any launch
        dvc.dvc_unet_decode_gop(net, lat, ctx, comm=c0)
    assert lib.dvc_comm_connect_local(c1.handle, c0.handle, c0.handle) != 0   # rank 1 of 2 has no successor
    assert lib.dvc_comm_connect_local(c0.handle, c0.handle, None) != 0        # next must be rank 1
    small = _net(dvc, torch.bfloat16, SMALL, 32, 8, 12, 4, 8)
    s0, s1 = dvc.Comm(0, 2, small, _connect=False), dvc.Comm(1, 2, small, _connect=False)
    dvc.check(lib.dvc_comm_connect_local(s0.handle, s1.handle, None))
    dvc.check(lib.dvc_comm_connect_local(s1.handle, None, s0.handle))
    with pytest.raises(dvc.DvcError):          # receive slots sized for a smaller network's carry
        dvc.dvc_unet_decode_gop(net, lat, ctx, comm=s0)


def _ipc_worker(rank, world, port, T, h, w, q):
    import torch.distributed as dist

    import paper_2601_20564_b200 as dvc
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dtype = torch.bfloat16
    net = _net(dvc, dtype, SMALL, 32, h, w, T, 8)
    comm = dvc.Comm(rank, world, net)          # IPC handles over torch.distributed
    a, b = dvc.chunk_bounds(T, world)[rank]
    res = []
    for call in range(3):
        lat, ctx = _inputs(T, h, w, 32, dtype, 30 + call)
        k = torch.zeros(net.carry_elems, dtype=dtype, device="cuda")
        out = dvc.dvc_unet_decode_gop(net, lat[a:b].contiguous(), ctx[a:b].contiguous(), comm=comm,
                                      carry_out=k if rank == world - 1 else None)
        torch.cuda.synchronize()
        res.append((out.cpu(), k.cpu()))
    dist.barrier()
    comm.close()
    q.put((rank, res))
    dist.destroy_process_group()


def test_ipc_halo_two_processes_equals_single_rank(dvc):
    import torch.multiprocessing as mp
    T, h, w, world = 6, 12, 20, 2
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    procs = [ctx_mp.Process(target=_ipc_worker, args=(r, world, 29611, T, h, w, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    try:
        for _ in range(world):
            r, res = q.get(timeout=300)
            got[r] = res
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    net = _net(dvc, torch.bfloat16, SMALL, 32, h, w, T, 8)
    for call in range(3):
        lat, ctx = _inputs(T, h, w, 32, torch.bfloat16, 30 + call)
        k = torch.zeros(net.carry_elems, dtype=torch.bfloat16, device="cuda")
        ref = dvc.dvc_unet_decode_gop(net, lat, ctx, carry_out=k).cpu()
        assert torch.equal(torch.cat([got[r][call][0] for r in range(world)]), ref), call
        assert torch.equal(got[world - 1][call][1], k.cpu()), call


def test_bench_multi_rank_path_on_one_gpu(dvc):
    """bench.py's N > 1 path end to end (torchrun re-launch, IPC handle exchange over the process group,
    P2P halo per ResBlock, max-over-ranks timing, e2e) with both ranks sharing cuda:0 (--share-device:
    gloo plumbing, since NCCL refuses two ranks on one GPU).  The throughput of time-sliced ranks means
    nothing; the line's shape and rc do."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if not k.startswith("DVC_") and k not in ("WORLD_SIZE", "RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--share-device", "--steps", "2",
                        "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True, timeout=600, env=env,
                       cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["config"]["frames_per_gpu"] == 16
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0


@pytest.mark.parametrize("h,w,T,world", [(90, 160, 8, 4), (135, 240, 6, 2)])
def test_loopback_halo_full_size(dvc, h, w, T, world):
    """G11 at the configs' latent sizes (720p headline, 1080p C4) and widths: the P2P halo between
    concurrent loopback ranks equals the single-rank decode bit for bit, carry_out included."""
    dtype = torch.bfloat16
    net = _net(dvc, dtype, (240, 480, 960, 960), 256, h, w, T, 24)
    comms = dvc.Comm.local_group(world, net)
    lat, ctx = _inputs(T, h, w, 256, dtype, 40)
    ref_k = torch.empty(net.carry_elems, dtype=dtype, device="cuda")
    ref = dvc.dvc_unet_decode_gop(net, lat, ctx, carry_out=ref_k)
    for _ in range(3):
        k = torch.zeros(net.carry_elems, dtype=dtype, device="cuda")
        assert torch.equal(_loopback(dvc, net, comms, lat, ctx, k), ref)
        assert torch.equal(k, ref_k)
