"""Host-side logic of the bench and of the multi-GPU split (-m "not gpu", CPU only):

* `bench.py --gpus 2 --dry-run` re-launches itself under torch.distributed.run with two ranks that
  rendezvous over gloo on 127.0.0.1 (the driver's N>1 launch path, without GPUs);
* the contiguous frame chunks of a GOP (the remainder goes to the last ranks) and
  the neighbour selection of the halo's handle exchange, over a real world-2 gloo all_gather;
* bench.py refuses to time anything with an experiment knob (DVC_*) in the environment.
"""
import json
import os
import subprocess
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env():
    return {k: v for k, v in os.environ.items() if not k.startswith("DVC_") and k not in ("WORLD_SIZE", "RANK")}


@pytest.mark.parametrize("n,scaling,chunks", [(2, "strong", [[0, 16], [16, 32]]),
                                              (3, "strong", [[0, 10], [10, 21], [21, 32]]),
                                              (2, "weak", [[0, 32], [0, 32]])])
def test_bench_self_launches_n_ranks(n, scaling, chunks):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--dry-run",
                        "--scaling", scaling], capture_output=True, text=True, timeout=240, env=_env(), cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == n and line["ranks"] == list(range(n)) and line["chunks"] == chunks


def test_bench_refuses_experiment_knobs():
    env = dict(_env(), DVC_FZ_XNOSTATS="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run"], capture_output=True,
                       text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode != 0 and "DVC_FZ_XNOSTATS" in r.stderr


def test_chunk_bounds():
    import paper_2601_20564_b200 as dvc
    assert dvc.chunk_bounds(32, 1) == [(0, 32)]
    assert dvc.chunk_bounds(32, 8) == [(4 * r, 4 * r + 4) for r in range(8)]
    assert dvc.chunk_bounds(5, 2) == [(0, 2), (2, 5)]
    for T in range(1, 20):
        for world in range(1, T + 1):
            b = dvc.chunk_bounds(T, world)
            sizes = [t1 - t0 for t0, t1 in b]
            assert b[0][0] == 0 and b[-1][1] == T and all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes)   # remainder on the last ranks
    with pytest.raises(ValueError):
        dvc.chunk_bounds(2, 3)


def _gather_worker(rank, world, port, q):
    import paper_2601_20564_b200 as dvc
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    handle = bytes([rank]) * 64                      # stands in for the 64-byte CUDA IPC handle
    gathered = [None] * world
    dist.all_gather_object(gathered, handle)
    q.put((rank, dvc.halo_neighbours(gathered, rank)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_handle_exchange_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, 29640 + world, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        nxt, prv = got[r]
        assert nxt == (bytes([r + 1]) * 64 if r < world - 1 else None)
        assert prv == (bytes([r - 1]) * 64 if r > 0 else None)
