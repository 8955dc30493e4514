"""Multi-process host logic of the sharded path on CPU (gloo, world_size 2).

The push itself needs a GPU; what N>1 adds on the host is covered here:
shard ranges, shard generation by global index, the per-step diagnostic
all_reduce(SUM) and the max-over-ranks timing."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2104_04579_b200.dist import shard_range


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 1000, 10_001, 800_000_003])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_ranges_tile_exactly(n, world):
    prev = 0
    for r in range(world):
        lo, hi = shard_range(n, r, world)
        assert lo == prev and lo <= hi
        if r < world - 1:
            assert hi % 8 == 0
        prev = hi
    assert prev == n


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import torch.distributed as dist
    import oracle
    import synth
    from paper_2104_04579_b200 import dist as bdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    bdist.init("gloo")
    w = synth.config("C5", n=n)
    lo, hi = shard_range(n, rank, world)
    d = w.generate(lo, hi - lo)
    pos = torch.stack([d["x"], d["y"], d["z"]], 1).numpy()
    mom = torch.stack([d["px"], d["py"], d["pz"]], 1).numpy()
    E = torch.stack([d["Ex"], d["Ey"], d["Ez"]], 1).numpy()
    B = torch.stack([d["Bx"], d["By"], d["Bz"]], 1).numpy()
    P, M, G = oracle.push(pos, mom, d["type"].numpy(), [w.types[0][0]], [w.types[0][1]],
                          w.light_velocity, oracle.FIELD_ARRAYS, E=E, B=B, dt=w.dt, n_steps=2)
    ke = oracle.kinetic_energy(M, G, d["weight"].numpy(), d["type"].numpy(), [w.types[0][1]],
                               w.light_velocity)
    diag = torch.tensor([ke, float(hi - lo)], dtype=torch.float64)
    bdist.allreduce_diag(diag)
    t = bdist.max_over_ranks(float(rank + 1) * 1.5)
    bdist.barrier()
    q.put((rank, diag.tolist(), t))
    dist.destroy_process_group()


def test_gloo_two_ranks_diag_allreduce():
    import oracle
    import synth
    n = 20_003
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # unsharded reference
    w = synth.config("C5", n=n)
    d = w.generate()
    pos = torch.stack([d["x"], d["y"], d["z"]], 1).numpy()
    mom = torch.stack([d["px"], d["py"], d["pz"]], 1).numpy()
    E = torch.stack([d["Ex"], d["Ey"], d["Ez"]], 1).numpy()
    B = torch.stack([d["Bx"], d["By"], d["Bz"]], 1).numpy()
    P, M, G = oracle.push(pos, mom, d["type"].numpy(), [w.types[0][0]], [w.types[0][1]],
                          w.light_velocity, oracle.FIELD_ARRAYS, E=E, B=B, dt=w.dt, n_steps=2)
    ke = oracle.kinetic_energy(M, G, d["weight"].numpy(), d["type"].numpy(), [w.types[0][1]],
                               w.light_velocity)
    for rank, diag, t in res:
        assert diag[1] == n
        assert diag[0] == pytest.approx(ke, rel=1e-13)
        assert t == 3.0


def test_shard_generation_equals_slice_of_whole():
    import synth
    w = synth.config("C5", n=5000)
    whole = w.generate()
    for r in range(3):
        lo, hi = shard_range(w.n, r, 3)
        part = w.generate(lo, hi - lo)
        for k in whole:
            assert torch.equal(part[k], whole[k][lo:hi]), k
