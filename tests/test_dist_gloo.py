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
