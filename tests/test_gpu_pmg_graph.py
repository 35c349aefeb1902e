"""precondition() as a CUDA-graph replay (pmg.graph = auto / on / off): between
two prepare() calls the V-cycles of the pMG preconditioner (the reference's
PmgContext.precondition, pmg.py:280-298) are a fixed launch sequence, so on
launch-bound meshes they are captured once and replayed.  The replay runs the
same kernels in the same order: everything below is bit for bit the eager
path, including whole time steps, and the non-physical fallback still fires."""

import numpy as np
import pytest
import torch

from paper_2202_09733_b200 import cases, pmg
from paper_2202_09733_b200 import time_integration as ti
from paper_2202_09733_b200.harness import ImplicitDriver
from paper_2202_09733_b200.spatial import Discretization

pytestmark = pytest.mark.gpu


def t(x):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device="cuda")


def _ctx(d, levels, smoother, graph, shift=50.0):
    return pmg.PmgContext(d, pmg.PmgPrecondConfig(pmg.PHierarchy.parse(levels, "2", smoother), smoother_shift=shift,
                                                  graph=graph))


@pytest.mark.parametrize("levels,smoother", [("3-2", "ej"), ("3-2-1", "ej"), ("3-2", "rk-ej")])
def test_replay_is_bitwise_the_eager_cycle(cuda, levels, smoother):
    c = cases.config(1)
    d = Discretization(c.mesh, c.p, c.eqn)
    rng = np.random.default_rng(3)
    ctxs = {g: _ctx(d, levels, smoother, g) for g in ("off", "on", "auto")}
    for rnd in range(3):   # every prepare() drops the graph; the cycle's arguments change
        q = t(c.q0 * (1.0 + 1e-3 * rnd * rng.standard_normal(c.q0.size)))
        for ctx in ctxs.values():
            ctx.prepare(q, 3.0 + rnd)
        for _ in range(4):
            X = t(rng.standard_normal(c.q0.size))
            Y = {g: ctx.precondition(X) for g, ctx in ctxs.items()}
            assert torch.equal(Y["off"], Y["on"]) and torch.equal(Y["off"], Y["auto"])
    assert ctxs["off"].graph_replays == 0
    # the first call of a context runs eagerly, then every call is a replay
    assert ctxs["on"].graph_replays == 3 * 4 - 1 and ctxs["auto"].graph_replays == 3 * 4 - 1


def test_output_survives_the_next_replay(cuda):
    c = cases.config(1)
    d = Discretization(c.mesh, c.p, c.eqn)
    ctx = _ctx(d, "3-2", "ej", "on")
    ctx.prepare(t(c.q0), 2.0)
    rng = np.random.default_rng(0)
    X1, X2 = t(rng.standard_normal(c.q0.size)), t(rng.standard_normal(c.q0.size))
    ctx.precondition(X1)
    Y1 = ctx.precondition(X1)
    keep = Y1.clone()
    ctx.precondition(X2)
    assert torch.equal(Y1, keep)


def test_numpy_in_numpy_out(cuda):
    c = cases.config(1)
    d = Discretization(c.mesh, c.p, c.eqn)
    on, off = _ctx(d, "3-2", "ej", "on"), _ctx(d, "3-2", "ej", "off")
    for ctx in (on, off):
        ctx.prepare(c.q0, 2.0)
    v = np.random.default_rng(1).standard_normal(c.q0.size)
    for _ in range(2):
        a, b = on.precondition(v), off.precondition(v)
        assert isinstance(a, np.ndarray) and np.array_equal(a, b)


def test_esdirk3_step_identical_with_and_without_graph(cuda):
    c = cases.config(1)
    d = Discretization(c.mesh, c.p, c.eqn)
    s = ti.get_scheme("esdirk3")
    out = {}
    for g in ("off", "on"):
        cfg = {"case.precond": "pmg", "pmg.levels": "3-2", "pmg.smooth": "2", "pmg.smoother_shift": 50.0,
               "gmres.kdim": 30, "gmres.rtol": 1e-3, "ptc.dtau_init": c.dt, "ptc.rtol": 1e-4, "pmg.graph": g}
        drv = ImplicitDriver(d, cfg)
        q1, info = drv.step(t(c.q0), c.dt, s)
        out[g] = (q1, [i["iters"] for i in info], [x for i in info for x in i["gmres_per_iter"]],
                  drv.ctx.graph_replays)
    assert torch.equal(out["off"][0], out["on"][0])
    assert out["off"][1:3] == out["on"][1:3]
    assert out["off"][3] == 0 and out["on"][3] > 50


def test_non_physical_fallback_under_replay(cuda):
    """A direction that drives the cycle's state non-physical: the status word
    is read after the replay and the EJ fallback (pmg.py:292-296) answers."""
    c = cases.config(1)
    d = Discretization(c.mesh, c.p, c.eqn)
    on, off = _ctx(d, "3-2", "ej", "on", shift=0.0), _ctx(d, "3-2", "ej", "off", shift=0.0)
    for ctx in (on, off):
        ctx.prepare(t(c.q0), 1e-3)
    rng = np.random.default_rng(5)
    good = t(rng.standard_normal(c.q0.size))
    bad = t(1e9 * rng.standard_normal(c.q0.size))
    for X in (good, bad, good, bad):
        a, b = on.precondition(X), off.precondition(X)
        assert torch.equal(a, b)
    assert on.fallbacks == off.fallbacks and on.fallbacks >= 2


def test_auto_is_off_on_large_meshes_and_with_mbnk(cuda):
    c = cases.config(1)
    d = Discretization(c.mesh, c.p, c.eqn)
    ctx = _ctx(d, "3-2", "ej", "auto")
    assert ctx._graphable()
    ctx.GRAPH_AUTO_DOFS = 100
    assert not ctx._graphable()
    assert not pmg.PmgContext(d, pmg.PmgPrecondConfig(pmg.PHierarchy.parse("3-2", "2", "mbnk"),
                                                      graph="on"))._graphable()
    with pytest.raises(ValueError):
        pmg.PmgPrecondConfig(pmg.PHierarchy.parse("3-2", "2"), graph="sometimes")
