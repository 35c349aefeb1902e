"""world_size-2 gloo test of the multi-rank bench path (replicas, max-over-
ranks timing), on the CPU with the oracle standing in for the device."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    from oracle.fr_oracle import OracleDisc
    from paper_2202_09733_b200 import cases, dist
    dist.init("gloo")
    c = cases.config(1, nx=4)
    d = OracleDisc(c.mesh, c.p, c.eqn)
    R = d.residual(c.q0)
    fake_time = 0.1 * (rank + 1)                 # rank 1 is the slow one
    tmax, = dist.max_over_ranks([fake_time])
    rate = dist.job_rate(d.n_dofs, world, tmax)
    # replicas compute identical residuals: check through a collective
    checksum, = dist.max_over_ranks([float(np.abs(R).sum())])
    out[rank] = (tmax, rate, checksum, float(np.abs(R).sum()))
    dist.barrier()


@pytest.mark.timeout(300)
def test_two_rank_replicas_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == pytest.approx(0.2)
    n = res[0][1] * 0.2 / world
    assert res[0][1] == res[1][1] and n == pytest.approx(4 * 4 * 16 * 4)
    assert res[0][2] == res[1][2] == res[0][3] == res[1][3]


def _halo_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    import torch
    from paper_2202_09733_b200 import dist
    from paper_2202_09733_b200.partition import SlabPartition
    dist.init("gloo")
    nx, ny, sz = 4, 3 * world, 7
    part = SlabPartition(nx, ny, 1.0, 1.0, world, rank)
    q_global = torch.from_numpy(np.random.default_rng(0).standard_normal(nx * ny * sz))
    q_local = torch.zeros(part.n_local * sz, dtype=torch.float64)
    o = part.owned
    q_local[o.start * sz:o.stop * sz] = part.scatter_global(q_global, sz)[o.start * sz:o.stop * sz]
    q_ag = q_local.clone()
    part.exchange(q_local, sz)
    part.exchange_allgather(q_ag, sz)
    out[rank] = bool(torch.equal(q_local, part.scatter_global(q_global, sz))) and bool(torch.equal(q_local, q_ag))
    dist.barrier()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_slab_halo_exchange_gloo(world):
    # the multi-GPU partitioned residual's only data-path exchange (two-
    # neighbour send/recv): every rank's halo rows must come back equal to
    # the global field there, and to the round-1 all_gather form
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_halo_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert all(res[r] for r in range(world))


@pytest.mark.parametrize("world", [1, 2, 4])
def test_slab_owned_residual_is_exact_oracle(world):
    # two halo rows make the owned rows' residual exact (BR1 reaches two
    # elements deep): oracle R on each strip == global R at those elements
    from oracle.fr_oracle import OracleDisc
    from paper_2202_09733_b200 import cases
    from paper_2202_09733_b200.partition import SlabPartition
    c = cases.config(2, nx=8)
    g = OracleDisc(c.mesh, c.p, c.eqn)
    Rg = g.residual(c.q0).reshape(-1, g.offsets[1])
    Q = c.q0.reshape(-1, g.offsets[1])
    for rank in range(world):
        part = SlabPartition(8, 8, 10.0, 10.0, world, rank)
        lo = OracleDisc(part.mesh, c.p, c.eqn)
        Rl = lo.residual(Q[part.global_elements].reshape(-1)).reshape(-1, g.offsets[1])
        own = part.global_elements[part.owned]
        assert np.max(np.abs(Rl[part.owned] - Rg[own])) <= 1e-13 * np.max(np.abs(Rg))


def _reduce_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    from paper_2202_09733_b200 import dist
    from paper_2202_09733_b200.partition import SlabPartition
    dist.init("gloo")
    part = SlabPartition(4, 2 * world, 1.0, 1.0, world, rank)
    s = part.allreduce(rank + 1.0, "sum")
    mx = part.allreduce(rank + 1.0, "max")
    # rank 1 sees a non-physical state in its first owned element, rank 0 in
    # a halo element (a global id owned by the last rank): every rank must
    # agree on the smallest global id
    loc = part.owned.start if rank == 1 else 0
    st = part.reduce_status(1, loc)
    none = part.reduce_status(0, 0)
    out[rank] = (s, mx, st, none, int(part.global_elements[loc]))
    dist.barrier()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_partition_reductions_gloo(world):
    # the partitioned solver's scalar collectives: owned-range sums, the
    # non-finite / any-nonzero max, and the status word (smallest
    # (kind, global element) over the ranks)
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_reduce_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    total = world * (world + 1) / 2
    gids = [res[r][4] for r in range(world) if r in (0, 1)]
    for r in range(world):
        s, mx, st, none, _ = res[r]
        assert s == total and mx == world
        assert st == (1, min(gids)) and none == (0, 0)
