#!/usr/bin/env python
"""Benchmark of the FP64 FR residual hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "config 2"): 256x256 periodic quad
mesh, p=4 (25 points/element), compressible Navier-Stokes, Roe + BR1
(SURVEY 8.0), isentropic vortex + seeded 1e-6 noise; 6,553,600 FP64 DoF.
A "step" is one residual evaluation R(q) over the whole mesh; value =
DoF-updates/s (GDoF/s) over all ranks.  Also timed: the fused Jv (the
GMRES matvec), BASELINE's Rusanov + LDG variant of the same R, ten
ESDIRK3 JFNK-pMG p{4-2} time steps at config 2 (the metric's second
half), config 1's step beside the CPU oracle, configs 3-5.

Multi-GPU (N > 1): the headline is the PARTITIONED residual -- rank r
owns a 256 x 256 slab of one 256 x 256N periodic mesh, and every timed
step is the two-neighbour halo exchange (NCCL send/recv straight into the
halo rows) + R on the rank's strip (paper_2202_09733_b200/partition.py,
DESIGN.md section 6).  The replica number (each rank its own config-2
mesh) is reported next to it.  At N = 1 the headline is the plain config-2
mesh.  Times are CUDA-event device times on the launching stream, max over
ranks.  The rank-0-only extras (steps, other configs, CPU baseline) run at
N = 1 only.

--impl reference: the reference arm -- the CPU oracle (NumPy restatement
of the reference, oracle/, pinned to the reference's golden vectors)
timed on all of this box's host cores (OracleDisc.residual_mt: element
chunks on a thread pool, bitwise equal to the serial oracle) on the same
config and metric.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "FP64 FR residual/Jv GDoF/s (% HBM roofline); JFNK-pMG wall time per time step"
UNIT = "GDoF/s"
FLOP_PER_DOF_R = {2: 190.2, 3: 185.6, 4: 186.8, 5: 191.0}   # instrumented reference count
BYTES_PER_DOF_R = 16.0                                          # read q + write R (compulsory)
BYTES_PER_DOF_JV = 32.0                                         # read q, v, R0; write out


def workload(case, config):
    """The config dict both arms print (identical strings: same_config)."""
    n1 = int(round(np.sqrt(case.mesh.n_elements)))
    return {"workload": f"config{config}: R(u) over {case.mesh.n_elements} elements ({n1}^2 periodic), "
                        f"p={case.p}, {case.n_dofs} DoF, NS Roe+BR1 (SURVEY 8.0)"}


def src_hash():
    """Hash of the CUDA sources: stamps the committed ncu traffic figure."""
    import hashlib
    h = hashlib.sha256()
    for f in sorted((ROOT / "paper_2202_09733_b200" / "csrc").glob("*.cu*")):
        h.update(f.read_bytes())
    return h.hexdigest()[:16]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-step", action="store_true", help="skip the JFNK-pMG time-step timings")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU-oracle baseline sample")
    ap.add_argument("--no-configs", action="store_true", help="skip the configs 3-5 measurements")
    ap.add_argument("--no-mbnk", action="store_true", help="skip the MBNK smoother timings")
    return ap.parse_args()


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle

def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_residual_rate(case, seconds_budget=20.0, max_calls=None, threads=None):
    """Time the oracle residual on this host: OracleDisc.residual_mt, the
    element-chunked phases of the NumPy oracle on a thread pool (bitwise
    equal to OracleDisc.residual, tests/test_oracle_golden.py)."""
    from oracle.fr_oracle import OracleDisc
    T = threads or host_threads()
    d = OracleDisc(case.mesh, case.p, case.eqn)
    d.residual_mt(case.q0, threads=T)  # warm caches + pool
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        d.residual_mt(case.q0, threads=T)
        times.append(time.perf_counter() - t0)
        if (max_calls and len(times) >= max_calls) or time.perf_counter() - t_start > seconds_budget:
            break
    best = min(times)
    return case.n_dofs / best / 1e9, best, len(times), T


def run_reference(args):
    ws, rank, _ = dist_info()
    if rank != 0:
        return 0
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle.fr_oracle import OracleDisc
    from paper_2202_09733_b200 import cases
    case = cases.config(args.config)
    d = OracleDisc(case.mesh, case.p, case.eqn)
    T = host_threads()
    for _ in range(max(0, args.warmup)):
        d.residual_mt(case.q0, threads=T)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        d.residual_mt(case.q0, threads=T)
    el = time.perf_counter() - t0
    rate = case.n_dofs * args.steps / el / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded isentropic vortex + 1e-6 noise, SURVEY 8(d))",
        "config": dict(workload(case, args.config), parallelism="cpu"),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": T, "kind": "port",
                         "sample": f"{args.steps} full-mesh residual evaluations of config{args.config} "
                                   f"by the NumPy oracle (oracle/fr_oracle.py residual_mt), {T} threads"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md clocks line)

class ClockSampler:
    """SM clock / throttle-reason samples over a whole measurement (NVML
    every 20 ms in a thread; nvidia-smi if NVML is unavailable)."""
    NV_REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                  "sw_power_cap": 0x4}

    def __init__(self, gpu_index, period=0.02):
        self.gpu, self.period = gpu_index, period
        self.sm, self.mx, self.reasons = [], [], []
        self._stop = threading.Event()
        self._thr = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv = self._nvml
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)))
        self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)))
        fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        mask = fn(self._h)
        self.reasons.append({k for k, bit in self.NV_REASONS.items() if mask & bit})

    def _sample_smi(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={fields}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        r = [c.strip() for c in out.split(",")]
        if len(r) >= 6 and r[0].replace(".", "").isdigit():
            self.sm.append(float(r[0]))
            self.mx.append(float(r[1]))
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            self.reasons.append({names[i] for i in range(4) if r[2 + i].lower().startswith("active")})

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample_nvml() if self._nvml else self._sample_smi()
            except Exception:
                pass
            self._stop.wait(self.period if self._nvml else 0.1)

    def __enter__(self):
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._thr.join(timeout=10)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx),
                "reasons": sorted(set().union(*self.reasons)), "samples": len(self.sm),
                "source": "NVML, 20 ms period, over every timed section" if self._nvml else "nvidia-smi"}


# ---------------------------------------------------------------------------
# our arm

def measure_fp64_peak(torch, lib, stream):
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    blocks, iters = 148 * 8, 20000
    lib.pmgb_probe_fp64(1000, blocks, out.data_ptr(), stream)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.pmgb_probe_fp64(iters, blocks, out.data_ptr(), stream)
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1) * 1e-3
        best = max(best, 2.0 * 8 * iters * blocks * 256 / t / 1e12)
    return best


def event_time(torch, fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(reps):
        fn(i)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e-3


def rotating(torch, case, disc, nbuf):
    q0 = torch.as_tensor(case.q0, device="cuda")
    n = disc.n_dofs
    qs = [q0.clone() for _ in range(nbuf)]
    Rs = [torch.empty_like(q0) for _ in range(nbuf)]
    Xs = [torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(i))
          for i in range(nbuf)]
    R0s = [disc.residual(q) for q in qs]
    return qs, Rs, Xs, R0s


def run_ours(args):
    import torch
    from paper_2202_09733_b200 import dist as pdist
    ws, rank, local = dist_info()
    torch.cuda.set_device(local)
    pdist.init("nccl", torch.device("cuda", local))
    from paper_2202_09733_b200 import _lib, cases
    from paper_2202_09733_b200.spatial import Discretization
    from paper_2202_09733_b200.vec import launch_count, stream

    lib = _lib.load()
    W = max(3, args.warmup)
    K = max(1, args.steps)
    case = cases.config(args.config)
    disc = Discretization(case.mesh, case.p, case.eqn)
    n = disc.n_dofs
    st = stream()
    measured = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = float(measured.get("hbm_gbs", 6650.0))
    clk = ClockSampler(local)
    clk.__enter__()
    fp64_peak = measure_fp64_peak(torch, lib, st)

    # plain config-2 mesh (the N = 1 headline; replicas at N > 1), 4
    # rotating q/R buffer pairs (4 x 105 MB > 126 MB L2)
    nbuf = 4
    qs, Rs, Xs, R0s = rotating(torch, case, disc, nbuf)

    def r_step(i):
        disc.eval(qs[i % nbuf], _lib.EPI_R, Rs[i % nbuf])

    def jv_step(i):
        j = i % nbuf
        disc.eval(qs[j], _lib.EPI_JV, Rs[j], X=Xs[j], eps=1e-6, s=3.7, R0=R0s[j])

    for i in range(W):
        r_step(i)
        jv_step(i)
    torch.cuda.synchronize()
    pdist.barrier()
    l0 = launch_count()
    t_r = event_time(torch, r_step, K)
    launches_r = launch_count() - l0
    t_jv = event_time(torch, jv_step, K)
    t_r, t_jv = pdist.max_over_ranks([t_r, t_jv], "cuda")
    rate_plain = pdist.job_rate(n * K, ws, t_r) / 1e9
    rate_jv = pdist.job_rate(n * K, ws, t_jv) / 1e9
    per_gpu_r = n / (t_r / K)
    per_gpu_jv = n / (t_jv / K)

    # the same R through the general (bilinear-element) kernels: A/B of the
    # rectangle path on this mesh
    path = disc.residual_path()
    general = None
    if path == "rect":
        disc.residual_path("general")
        for i in range(W):
            r_step(i)
        t_g = event_time(torch, r_step, K)
        t_g, = pdist.max_over_ranks([t_g], "cuda")
        general = {"r_gdofs": pdist.job_rate(n * K, ws, t_g) / 1e9, "r_ms": t_g / K * 1e3,
                   "kernels": "k_trace_lines + k_fvn + k_assemble_async (csrc/fr_kernels.cu)"}
        disc.residual_path("rect")

    # e2e through the public API with host buffers: every step copies its q
    # from pinned host memory, evaluates R and copies R back; the
    # Discretization.residual_batch call overlaps step i's H2D, step i-1's
    # compute and step i-2's D2H on two copy engines + the compute stream.
    qh = [torch.from_numpy(case.q0.copy()).pin_memory() for _ in range(2)]
    Rh = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
    disc.residual_batch([qh[i % 2] for i in range(W)], [Rh[i % 2] for i in range(W)])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    disc.residual_batch([qh[i % 2] for i in range(K)], [Rh[i % 2] for i in range(K)])
    e1.record()
    e1.synchronize()
    t_e2e = e0.elapsed_time(e1) * 1e-3
    t_e2e, = pdist.max_over_ranks([t_e2e], "cuda")
    rate_e2e = pdist.job_rate(n * K, ws, t_e2e) / 1e9
    e2e_ok = bool(np.array_equal(Rh[(K - 1) % 2].numpy(), disc.residual(qs[0]).cpu().numpy()))
    # the e2e ceiling: one step's H2D and D2H copies running concurrently
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    dq, dR = torch.empty_like(qs[0]), torch.empty_like(qs[0])

    def duplex(i):
        with torch.cuda.stream(s_in):
            dq.copy_(qh[i % 2], non_blocking=True)
        with torch.cuda.stream(s_out):
            Rh[i % 2].copy_(dR, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s_in)
        torch.cuda.current_stream().wait_stream(s_out)
    for i in range(3):
        duplex(i)
    t_dup = event_time(torch, duplex, K)
    t_dup, = pdist.max_over_ranks([t_dup], "cuda")
    ceil_e2e = pdist.job_rate(n * K, ws, t_dup) / 1e9
    del qs, Rs, Xs, R0s
    torch.cuda.empty_cache()

    # the sharded residual with its halo exchange (all ranks take part); an
    # error on any rank is all-reduced so every rank leaves together
    try:
        partitioned = time_partitioned(torch, case, K, W, ws, rank, args.no_step or ws > 1)
        err = 0.0
    except Exception as exc:  # pragma: no cover
        partitioned = {"error": str(exc)[:200]}
        err = 1.0
    if max(pdist.max_over_ranks([err], "cuda")) > 0 and "error" not in partitioned:
        partitioned = {"error": "another rank failed"}

    # rank-0 extras (single GPU only: ranks > 0 would wait in a collective)
    step, others, mbnk = {}, {}, {}
    if ws == 1:
        if not args.no_step:
            step = time_steps(torch, case, args)
        if not args.no_configs and args.config == 2:
            others = time_other_configs(torch, args)
            others["config2_rusanov_ldg"] = time_variant_r(torch, case, K, W, riemann="rusanov",
                                                           viscous_scheme="ldg")
        if not args.no_mbnk and args.config == 2:
            try:
                mbnk = time_mbnk(torch, case)
            except Exception as exc:  # pragma: no cover
                mbnk = {"error": str(exc)[:200]}
    clk.__exit__()

    if rank != 0:
        pdist.barrier()
        return 0

    if ws > 1 and "r_gdofs" in partitioned:
        value, ms = partitioned["r_gdofs"], partitioned["ms_per_step"]
        parallelism = f"dp{ws}: partitioned 256 x {256 * ws} mesh, halo send/recv per step (NCCL)"
    else:
        value, ms = rate_plain, t_r / K * 1e3
        parallelism = "single GPU"
    flops = FLOP_PER_DOF_R[case.p] * n
    achieved = flops / (t_r / K) / 1e12
    flops_jv = (FLOP_PER_DOF_R[case.p] + 4.0) * n
    achieved_jv = flops_jv / (t_jv / K) / 1e12
    kern = ("R(u): k_rgf + k_rasm (csrc/fr_rect.cu)" if path == "rect"
            else "R(u): k_trace_lines + k_fvn + k_assemble_async (csrc/fr_kernels.cu)")
    cfg = dict(workload(case, args.config), l2="4 rotating q/R buffer pairs (419 MB > 126 MB L2)",
               parallelism=parallelism, residual_path=path)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": W,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded isentropic vortex + 1e-6 noise, SURVEY 8(d))",
        "config": cfg,
        "single_mesh": {"r_gdofs": rate_plain, "r_ms": t_r / K * 1e3,
                        "what": "each rank its own config-2 mesh (replicas)" if ws > 1 else "config-2 mesh"},
        "jv_gdofs": rate_jv,
        "jv_ms": t_jv / K * 1e3,
        "general_kernels": general,
        "roofline": {
            "bound": "fp64", "kernel": kern,
            "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
            "peak_source": "measured in this run (DFMA probe, pmgb_probe_fp64; MEASURED_PEAKS.json has no FP64)",
            "flop_per_dof": FLOP_PER_DOF_R[case.p],
            "hbm_view": {"achieved_gbs": BYTES_PER_DOF_R * per_gpu_r / 1e9, "peak_gbs": hbm_peak,
                         "frac": BYTES_PER_DOF_R * per_gpu_r / 1e9 / hbm_peak,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
            "bound_gdofs": min(hbm_peak / BYTES_PER_DOF_R, fp64_peak * 1e3 / FLOP_PER_DOF_R[case.p]),
            "traffic": None,
        },
        "roofline_jv": {
            "bound": "balanced (fp64 and hbm)", "achieved_tflops": achieved_jv, "fp64_frac": achieved_jv / fp64_peak,
            "flop_per_dof": FLOP_PER_DOF_R[case.p] + 4.0, "bytes_per_dof": BYTES_PER_DOF_JV,
            "achieved_gbs": BYTES_PER_DOF_JV * per_gpu_jv / 1e9,
            "hbm_frac": BYTES_PER_DOF_JV * per_gpu_jv / 1e9 / hbm_peak,
            "bound_gdofs": min(hbm_peak / BYTES_PER_DOF_JV, fp64_peak * 1e3 / (FLOP_PER_DOF_R[case.p] + 4.0)),
        },
        "e2e": {"value": rate_e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                "api": "Discretization.residual_batch (pinned host in/out, copies overlapped with compute)",
                "matches_device_path": e2e_ok,
                "pcie_ceiling": {"value": ceil_e2e, "unit": UNIT, "frac": rate_e2e / ceil_e2e,
                                 "what": "the step's H2D and D2H copies alone, concurrently (no compute)"}},
        "gpu_launches": int(launches_r),
        "clocks": clk.summary(),
        "step_time": step,
        "configs": others,
        "mbnk": mbnk,
        "partitioned": partitioned,
    }
    # CPU baseline: the oracle on this host, bounded sample
    try:
        if args.no_cpu or ws > 1:
            raise RuntimeError("skipped (--no-cpu or N > 1)")
        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
        cpu_rate, best, ncall, T = cpu_residual_rate(case, seconds_budget=15.0)
        line["cpu_baseline"] = {"value": cpu_rate, "unit": UNIT, "cores": T, "kind": "port",
                                "sample": f"best of {ncall} full-mesh oracle residual evaluations "
                                          f"(config{args.config}, residual_mt on {T} threads, {best:.2f} s each)"}
    except Exception as exc:  # pragma: no cover
        line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "port", "sample": f"{exc}"}
    # ncu DRAM bytes of one R, from the committed capture of the same kernel
    # sources (stamped with their hash; "stale" if the kernels changed since)
    prof = ROOT / "profiles" / "traffic_r2.json"
    if prof.exists():
        try:
            tr = json.loads(prof.read_text())
            line["roofline"]["traffic"] = tr.get(f"config{args.config}_R_bytes")
            line["roofline"]["traffic_source"] = {"file": "profiles/traffic_r2.json",
                                                  "sources_match": tr.get("src_hash") == src_hash()}
        except Exception:
            pass
    print(json.dumps(line), flush=True)
    pdist.barrier()
    return 0


def time_variant_r(torch, case, K, W, **eqn_changes):
    """R rate of the config-2 mesh with other EquationSpec options
    (BASELINE's literal Rusanov + LDG; parity unpinned)."""
    import dataclasses

    from paper_2202_09733_b200 import _lib
    from paper_2202_09733_b200.spatial import Discretization
    try:
        eqn = dataclasses.replace(case.eqn, **eqn_changes)
        d = Discretization(case.mesh, case.p, eqn)
        nb = 4
        q0 = torch.as_tensor(case.q0, device="cuda")
        qs = [q0.clone() for _ in range(nb)]
        Rs = [torch.empty_like(q0) for _ in range(nb)]
        step = lambda i: d.eval(qs[i % nb], _lib.EPI_R, Rs[i % nb])  # noqa: E731
        for i in range(W):
            step(i)
        t = event_time(torch, step, K)
        rec = {"options": eqn_changes, "r_gdofs": d.n_dofs * K / t / 1e9, "r_ms": t / K * 1e3,
               "residual_path": d.residual_path()}
        del d, qs, Rs
        torch.cuda.empty_cache()
        return rec
    except Exception as exc:  # pragma: no cover
        return {"options": eqn_changes, "error": str(exc)[:200]}


def time_other_configs(torch, args):
    """BASELINE configs 3-5: R and Jv rates (rotating
    buffers, >= 4x L2), config 3's nonlinear pMG solve per outer iteration
    (one V-cycle each, levels 4-3-2-1-0), config 4's ROW4 step (walls,
    GMRES(60), pMG 3-2), config 5 at capacity (151M DoF, R/Jv only:
    its p=5 EJ blocks would need 174 GB)."""
    from paper_2202_09733_b200 import _lib, cases, newton_krylov as nk, pmg
    from paper_2202_09733_b200 import time_integration as ti
    from paper_2202_09733_b200.harness import ImplicitDriver
    from paper_2202_09733_b200.spatial import Discretization
    out = {}
    for k in (3, 4, 5):
        rec = {}
        try:
            c = cases.config(k)
            d = Discretization(c.mesh, c.p, c.eqn)
            n = d.n_dofs
            nb = max(2, int(np.ceil(4 * 126e6 / (32.0 * n))))
            q0 = torch.as_tensor(c.q0, device="cuda")
            qs = [q0.clone() for _ in range(nb)]
            Rs = [torch.empty_like(q0) for _ in range(nb)]
            X = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(7))
            R0 = d.residual(q0)
            reps = 10 if n > 1e8 else 40
            r_step = lambda i: d.eval(qs[i % nb], _lib.EPI_R, Rs[i % nb])
            jv_step = lambda i: d.eval(qs[i % nb], _lib.EPI_JV, Rs[i % nb], X=X, eps=1e-6, s=3.7, R0=R0)
            for i in range(3):
                r_step(i)
                jv_step(i)
            t_r = event_time(torch, r_step, reps)
            t_jv = event_time(torch, jv_step, reps)
            rec.update(n_dofs=n, p=c.p, r_gdofs=n * reps / t_r / 1e9, r_ms=t_r / reps * 1e3,
                       jv_gdofs=n * reps / t_jv / 1e9, rotating_pairs=nb)
            del qs, Rs
            if k == 3:
                # EJ on every level (reference smoothers) and BASELINE's
                # pseudo-time RK on the levels above p=0 with EJ at p=0
                for key, sm in (("pmg_solve", "ej"), ("pmg_solve_rk", "rk-rk-rk-rk-ej")):
                    hier = pmg.PHierarchy.parse(c.levels, "2", sm)
                    ctx = pmg.PmgContext(d, pmg.PmgPrecondConfig(hier, smoother_shift=c.extra["smoother_shift"]))
                    pmg.pmg_solve(ctx, q0, nk.PtcConfig(dtau_init=0.1, max_iters=1, rtol=1e-14))
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    _, stt = pmg.pmg_solve(ctx, q0, nk.PtcConfig(dtau_init=0.1, max_iters=3, rtol=1e-14))
                    torch.cuda.synchronize()
                    el = time.perf_counter() - t0
                    rec[key] = {"levels": c.levels, "smoothers": sm, "outer_iters": stt["iters"], "s": el,
                                "ms_per_outer_iter_incl_prepare": el / max(1, stt["iters"]) * 1e3,
                                "rel_history": [h[1] for h in stt["history"]]}
                    del ctx
            if k == 4:
                cfg = {"case.precond": "pmg", "pmg.levels": c.levels, "pmg.smooth": "2",
                       "pmg.smoother_shift": c.extra["smoother_shift"], "gmres.kdim": c.kdim, "gmres.rtol": 1e-3}
                # ros4l: BASELINE's 4-stage ROW; row4: the reference's 6-stage
                # RODASP; both at the case dt (0.125 dt_conv, cases.py)
                for name, dt in ((c.scheme, c.dt), ("row4", c.dt)):
                    sch = ti.get_scheme(name)
                    try:
                        ImplicitDriver(d, cfg).step(q0, dt, sch)
                        drv = ImplicitDriver(d, cfg)
                        torch.cuda.synchronize()
                        t0 = time.perf_counter()
                        _, info = drv.step(q0, dt, sch)
                        torch.cuda.synchronize()
                        rec[f"{name}_step"] = {"s": time.perf_counter() - t0, "dt": dt, "stages": sch.stages,
                                               "gmres_iters": [i["iters"] for i in info]}
                    except Exception as exc:  # pragma: no cover
                        rec[f"{name}_step"] = {"dt": dt, "error": str(exc)[:200]}
                del drv
            del d, q0, X, R0
        except Exception as exc:  # pragma: no cover
            rec["error"] = str(exc)[:200]
        torch.cuda.empty_cache()
        out[f"config{k}"] = rec
    return out


def time_partitioned(torch, case2, K, W, ws, rank, no_step=False):
    """The sharded residual: rank r owns a 256 x 256 slab of a
    256 x 256N periodic box (the config-2 field on every slab, which is
    y-periodic) plus 2 halo element rows each side; every step is the
    two-neighbour halo exchange (NCCL send/recv into the halo rows) + R on
    the local strip.  Owned DoF per second over all ranks, device time max
    over ranks; halo bytes per rank and step reported."""
    from paper_2202_09733_b200 import dist as pdist
    from paper_2202_09733_b200.partition import PartitionedResidual, SlabPartition
    n1 = int(round(np.sqrt(case2.mesh.n_elements)))
    part = SlabPartition(n1, n1 * ws, 10.0, 10.0 * ws, ws, rank)
    pr = PartitionedResidual(part, case2.p, case2.eqn)
    sz = pr.sz
    pr.q_owned.copy_(torch.as_tensor(case2.q0, device="cuda"))
    out = torch.empty_like(pr.q_local)
    step = lambda i: pr.residual(out)
    xchg = lambda i: part.exchange(pr.q_local, sz)
    for i in range(W):
        step(i)
    torch.cuda.synchronize()
    pdist.barrier()
    t_r = event_time(torch, step, K)
    pdist.barrier()
    t_x = event_time(torch, xchg, K)
    t_r, t_x = pdist.max_over_ranks([t_r, t_x], "cuda")
    owned = part.rows * n1 * sz
    halo_bytes = 2 * 2 * part.halo * n1 * sz * 8  # sent + received, both sides
    rec = {"global_mesh": f"{n1} x {n1 * ws} periodic, {ws} slab(s) of {n1} x {n1}", "halo_rows": part.halo,
           "collective": "send/recv of 2 halo rows to each neighbour (NCCL, batch_isend_irecv)" if ws > 1
           else "local wrap copy",
           "r_gdofs": owned * K * ws / t_r / 1e9, "ms_per_step": t_r / K * 1e3,
           "exchange_ms": t_x / K * 1e3, "halo_bytes_per_rank_step": halo_bytes if ws > 1 else 0,
           "local_dofs_per_rank": pr.disc.n_dofs, "owned_dofs_per_rank": owned,
           "residual_path": pr.disc.residual_path()}
    del pr, out
    if no_step:
        return rec
    try:
        rec["solver_step"] = time_partitioned_step(torch, ws, rank)
    except Exception as exc:  # pragma: no cover
        rec["solver_step"] = {"error": str(exc)[:200]}
    return rec


def time_partitioned_step(torch, ws, rank):
    """The partitioned JFNK-pMG solver (partition.HaloDiscretization):
    config-1 physics, one ESDIRK3 step with pMG p{3-2} EJ, every rank a
    16 x 16 slab of a 16 x 16N periodic box (the config-1 field on every
    slab), halo refresh before every neighbour-reading kernel and
    owned-range reductions all-reduced over the ranks."""
    from paper_2202_09733_b200 import cases, dist as pdist, vec
    from paper_2202_09733_b200 import time_integration as ti
    from paper_2202_09733_b200.harness import ImplicitDriver
    from paper_2202_09733_b200.partition import HaloDiscretization, SlabPartition
    c = cases.config(1)
    part = SlabPartition(16, 16 * ws, 10.0, 10.0 * ws, ws, rank)
    d = HaloDiscretization(part, c.p, c.eqn)
    q0 = torch.zeros(d.n_dofs, dtype=torch.float64, device="cuda")
    vec.set_partition(part)
    try:
        vec.owned(q0).copy_(torch.as_tensor(c.q0, device="cuda"))
        cfg = {"case.precond": "pmg", "pmg.levels": c.levels, "pmg.smooth": "2", "pmg.smoother_shift": 50.0,
               "gmres.kdim": c.kdim, "gmres.rtol": 1e-3, "ptc.dtau_init": c.dt, "ptc.rtol": 1e-4}
        sch = ti.get_scheme(c.scheme)
        ImplicitDriver(d, cfg).step(q0, c.dt, sch)
        drv = ImplicitDriver(d, cfg)
        torch.cuda.synchronize()
        pdist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, info = drv.step(q0, c.dt, sch)
        e1.record()
        torch.cuda.synchronize()
        t, = pdist.max_over_ranks([e0.elapsed_time(e1) * 1e-3], "cuda")
    finally:
        vec.set_partition(None)
    return {"scheme": c.scheme, "pmg": c.levels, "global_mesh": f"16 x {16 * ws}", "s": t,
            "ptc_iters": [i["iters"] for i in info], "gmres_iters": [i["gmres_iters"] for i in info],
            "collectives": "halo all_gather per R + all_reduce per dot (NCCL)" if ws > 1 else "local"}


def time_mbnk(torch, case2):
    """MBNK smoother pieces on config 2's p=2 coarse
    level (65,536 elements, 327,680 36x36 blocks): block-sparse FD Jacobian,
    level-scheduled block ILU0 factor / apply, block SpMV."""
    from paper_2202_09733_b200 import cases, newton_krylov as nk, pmg
    from paper_2202_09733_b200.spatial import Discretization
    d4 = Discretization(case2.mesh, 4, case2.eqn)
    ctx = pmg.PmgContext(d4, pmg.PmgPrecondConfig(pmg.PHierarchy.parse("4-2")))
    qc = ctx.tables[0].restrict(torch.as_tensor(case2.q0, device="cuda"))
    dc = ctx.levels[1].disc
    nk.sparse_pattern(dc)

    def wall(fn, n=1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            r = fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / n, r
    nk.ilu0_factor(nk.assemble_sparse_blocks(dc, qc, 40.0))  # first calls load the kernels
    t_a, A = wall(lambda: nk.assemble_sparse_blocks(dc, qc, 40.0))
    t_f, F = wall(lambda: nk.ilu0_factor(A))
    v = torch.randn(dc.n_dofs, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    nk.ilu0_apply(F, v)
    t_ap, _ = wall(lambda: nk.ilu0_apply(F, v), 5)
    t_mv, _ = wall(lambda: A.matvec(v), 20)
    pat = A.pattern
    out = {"level": "config2 coarse p=2", "n_elements": dc.mesh.n_elements, "nnz_blocks": pat.nnz,
           "block": dc.elem_size, "ilu_levels": [len(pat.lo_ptr) - 1, len(pat.up_ptr) - 1],
           "assemble_ms": t_a * 1e3, "ilu0_factor_ms": t_f * 1e3, "ilu0_apply_ms": t_ap * 1e3,
           "spmv_ms": t_mv * 1e3, "timing": "wall clock around synchronised calls"}
    del A, F, ctx
    torch.cuda.empty_cache()
    return out


def time_steps(torch, case2, args):
    """JFNK-pMG time steps (after one warm-up step each): config 1 (one
    ESDIRK3 step, beside the CPU oracle's same step) and config 2 (BASELINE's
    ten ESDIRK3 steps with the reference's EJ smoothers in FP64, marching
    the solution; one step with the pseudo-transient RK smoother on the fine
    level -- north star item 3 -- and one with FP32-stored EJ factors).
    Step times are CUDA-event times on the solver's stream."""
    from paper_2202_09733_b200 import cases
    from paper_2202_09733_b200 import time_integration as ti
    from paper_2202_09733_b200.harness import ImplicitDriver
    from paper_2202_09733_b200.spatial import Discretization
    out = {}
    c1 = cases.config(1)
    # config2_fp32: pmg.block_precision = fp32 (FP32-stored EJ factors, FP64
    # arithmetic; not in the reference) -- the EJ apply is the step's top kernel
    runs = (("config1", c1, "ej-ej", "fp64"), ("config2", case2, "ej-ej", "fp64"),
            ("config2_rk", case2, "rk-ej", "fp64"), ("config2_fp32", case2, "ej-ej", "fp32"))
    discs = {}
    for key, c, smoothers, prec in runs:
        d = discs.setdefault(c.name, Discretization(c.mesh, c.p, c.eqn))
        cfg = {"case.precond": "pmg", "pmg.levels": c.levels, "pmg.smooth": "2", "pmg.smoother": smoothers,
               "pmg.smoother_shift": c.extra["smoother_shift"], "gmres.kdim": c.kdim,
               "gmres.rtol": 1e-3, "ptc.dtau_init": c.dt, "ptc.rtol": 1e-4, "pmg.block_precision": prec}
        q = torch.as_tensor(c.q0, device="cuda")
        sch = ti.get_scheme(c.scheme)
        rec = {"scheme": c.scheme, "pmg": c.levels, "smoothers": smoothers, "block_precision": prec,
               "smoother_shift": c.extra["smoother_shift"], "dt": c.dt}
        nsteps = c.steps if key == "config2" else 1
        try:
            drv = ImplicitDriver(d, cfg)
            drv.step(q, c.dt, sch)  # warm-up (allocator + caches)
            torch.cuda.synchronize()
            torch.cuda.reset_peak_memory_stats()
            drv = ImplicitDriver(d, cfg)
            times, ptc, gm = [], [], []
            for _ in range(nsteps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                q, info = drv.step(q, c.dt, sch)
                e1.record()
                e1.synchronize()
                times.append(e0.elapsed_time(e1) * 1e-3)
                ptc.append([i["iters"] for i in info])
                gm.append([i["gmres_iters"] for i in info])
            rec.update(gpu_s=statistics.mean(times), steps=nsteps, step_s=times, ptc_iters=ptc if nsteps > 1 else ptc[0],
                       gmres_iters=gm if nsteps > 1 else gm[0],
                       peak_device_gb=torch.cuda.max_memory_allocated() / 1e9)
            del drv
        except Exception as exc:
            rec.update(gpu_s=None, error=str(exc)[:200])
        torch.cuda.empty_cache()
        out[key] = rec
    try:
        from oracle import solver_oracle as so
        from oracle.fr_oracle import OracleDisc
        od = OracleDisc(c1.mesh, c1.p, c1.eqn)
        drv = so.Driver(od, "pmg", c1.levels, 2, smoother_shift=50.0, gmres_rtol=1e-3, dtau_init=c1.dt)
        s = ti.get_scheme(c1.scheme)
        t0 = time.perf_counter()
        drv.esdirk_step(c1.q0, c1.dt, s.a, s.b)
        out["config1"]["cpu_oracle_s"] = time.perf_counter() - t0
        out["config1"]["cpu_oracle_gmres_iters"] = [r[2] for r in drv.records]
        out["config1"]["speedup_vs_cpu"] = out["config1"]["cpu_oracle_s"] / out["config1"]["gpu_s"]
    except Exception as exc:  # pragma: no cover
        out["config1"]["cpu_oracle_s"] = f"failed: {exc}"
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
