"""Multi-rank plumbing for the replica (weak-scaling) bench path.

The north-star path is evaluated per mesh; BASELINE's multi-GPU runs are
independent replicas of the config-2 mesh, one per rank, with no
data-path collective.  The only cross-rank traffic
is the timing reduction: every rank times its own steps with CUDA events
and the job reports the MAX over ranks.  Backend "nccl" on GPUs, "gloo"
in the CPU tests; rendezvous through MASTER_ADDR/MASTER_PORT (127.0.0.1).
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str, device=None):
    ws, _, _ = env()
    if ws > 1 and not dist.is_initialized():
        kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
        dist.init_process_group(backend, **kw)
    return ws


def max_over_ranks(values, device="cpu"):
    """Element-wise max of a list of floats over all ranks."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [float(v) for v in values]
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def job_rate(units_per_rank: int, world: int, seconds_max: float) -> float:
    """Whole-job throughput: all ranks' units over the slowest rank's time."""
    return units_per_rank * world / seconds_max


def barrier():
    if dist.is_available() and dist.is_initialized():
        dist.barrier()
