"""Multi-GPU plumbing for bench.py (one process per GPU, torch.distributed).

* The decode step has no collective: every rank runs its own node replica;
  whole-job throughput = sum of rank tokens / max over ranks of device time.
* The disaggregated engine (P/D nodes on different GPUs, P->D KV hops over
  NVLink with ppd_kv_copy) runs in ONE process that drives all GPUs of the box
  (node i -> GPU i): rank 0 runs it while the other ranks wait at a barrier.
  node_layouts() names the P/D shapes measured at each GPU count (BASELINE
  configs[2..4]).
"""
from __future__ import annotations

import os

LAYOUTS = {1: ["1R"], 2: ["1P_1D"], 4: ["1P_3D", "2P_2D"], 8: ["2P_6D", "4P_4D"]}


def node_layouts(n_gpus: int) -> list[str]:
    if n_gpus in LAYOUTS:
        return LAYOUTS[n_gpus]
    if n_gpus >= 2:
        return [f"1P_{n_gpus - 1}D"]
    return ["1R"]


def layout_gpus(layout: str, n_gpus: int) -> list[int]:
    """Node i -> GPU i (P first, then D, then R, reference simulator.cpp:139-141)."""
    n_nodes = sum(int(p[:-1]) for p in layout.split("_"))
    if n_nodes > n_gpus:
        raise ValueError(f"{layout} needs {n_nodes} GPUs, have {n_gpus}")
    return list(range(n_nodes))


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (identity when not distributed)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(values)
    t = torch.tensor(values, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def sum_over_ranks(values, device=None):
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(values)
    t = torch.tensor(values, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.tolist()


def whole_job_throughput(rank_units: float, rank_time_s: float, device=None) -> float:
    """value = units all ranks processed / max over ranks of the timed region."""
    (units,) = sum_over_ranks([rank_units], device)
    (t,) = max_over_ranks([rank_time_s], device)
    return units / t
