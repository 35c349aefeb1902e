"""Element-partitioned JFNK-pMG step: slab strips with two
halo rows, halo refresh before every neighbour-reading kernel, owned-range
reductions summed over the ranks (partition.HaloDiscretization +
vec.set_partition).

World size 1 runs the whole plumbing with the local wrap exchange; world
size 2 runs two processes on the one GPU with the gloo backend (host-staged
collectives: a correctness test of the exchange and reduction path, not a
performance stand-in).  Each rank's owned rows must follow the single-mesh
step: same PTC counts, GMRES counts +-1 (the rank-split sums round
differently), solution within 1e-7."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CFG = {"case.precond": "pmg", "pmg.levels": "3-2", "pmg.smooth": "2", "pmg.smoother_shift": 50.0,
       "gmres.kdim": 30, "gmres.rtol": 1e-3, "ptc.rtol": 1e-4}


def _step(disc, q0, c, scheme, smoother, ortho="mgs"):
    from paper_2202_09733_b200 import time_integration as ti
    from paper_2202_09733_b200.harness import ImplicitDriver
    cfg = dict(CFG, **{"ptc.dtau_init": c.dt, "pmg.smoother": smoother, "gmres.ortho": ortho})
    q1, info = ImplicitDriver(disc, cfg).step(torch.as_tensor(q0, device="cuda"), c.dt, ti.get_scheme(scheme))
    return q1, [i.get("iters") for i in info], [i.get("gmres_iters", i.get("iters")) for i in info]


def _reference(scheme, smoother, ortho="mgs"):
    from paper_2202_09733_b200 import cases
    from paper_2202_09733_b200.spatial import Discretization
    c = cases.config(1)
    d = Discretization(c.mesh, c.p, c.eqn)
    q1, ptc, gm = _step(d, c.q0, c, scheme, smoother, ortho)
    return c, q1.cpu().numpy(), ptc, gm


def _rank_step(world, rank, scheme, smoother, ortho="mgs"):
    from paper_2202_09733_b200 import cases, vec
    from paper_2202_09733_b200.partition import HaloDiscretization, SlabPartition
    c = cases.config(1)
    part = SlabPartition(16, 16, 10.0, 10.0, world, rank)
    d = HaloDiscretization(part, c.p, c.eqn)
    sz = d.elem_size
    q0 = part.scatter_global(c.q0, sz)
    vec.set_partition(part)
    try:
        q1, ptc, gm = _step(d, q0, c, scheme, smoother, ortho)
        own = vec.owned(q1).cpu().numpy()
    finally:
        vec.set_partition(None)
    return part.global_elements[part.owned], own, ptc, gm


def _compare(c, ref, parts, ptc_ref, gm_ref):
    sz = c.q0.size // c.mesh.n_elements
    got = np.full(c.q0.size, np.nan)
    for ge, own, ptc, gm in parts:
        got.reshape(-1, sz)[ge] = own.reshape(-1, sz)
        assert ptc == ptc_ref, (ptc, ptc_ref)
        assert len(gm) == len(gm_ref) and all(abs(a - b) <= 1 for a, b in zip(gm, gm_ref)), (gm, gm_ref)
    assert not np.isnan(got).any()
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) <= 1e-7


@pytest.mark.parametrize("scheme,smoother,ortho", [("esdirk3", "ej-ej", "mgs"), ("ros4l", "rk-ej", "mgs"),
                                                   ("esdirk3", "ej-ej", "cgs2")])
def test_partitioned_step_one_rank(cuda, scheme, smoother, ortho):
    c, ref, ptc_ref, gm_ref = _reference(scheme, smoother, ortho)
    _compare(c, ref, [_rank_step(1, 0, scheme, smoother, ortho)], ptc_ref, gm_ref)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out, ortho="mgs"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    import torch.distributed as dist
    dist.init_process_group("gloo")
    try:
        ge, own, ptc, gm = _rank_step(world, rank, "esdirk3", "ej-ej", ortho)
        out[rank] = (ge, own, ptc, gm)
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.timeout(900)
@pytest.mark.parametrize("ortho", ["mgs", "cgs2"])
def test_partitioned_step_two_ranks_gloo(cuda, ortho):
    # cgs2: 3 all-reduces per Arnoldi step instead of j + 2
    import torch.multiprocessing as mp
    c, ref, ptc_ref, gm_ref = _reference("esdirk3", "ej-ej", ortho)
    world, port = 2, _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out, ortho), nprocs=world, join=True)
        parts = [out[r] for r in range(world)]
    _compare(c, ref, parts, ptc_ref, gm_ref)
