"""Multi-GPU host logic: one process per GPU, torch.distributed for plumbing.

Two decompositions:

* **Probe sharding** (used by bench.py at N>1): Hessian applies on different
  vectors are independent units, so each rank applies H̃ to its own
  contiguous shard of probes with no data-path collective; the job time is
  the maximum over ranks ("scaling": "weak").
* **Spectral-row sharding** (large n_x): in the DST eigenbasis the
  sweep recurrence is pointwise, so the rows (spectral modes) of every
  n_x-tall factor split across ranks with NO halo; the only exchanges are the
  small per-flush partial sums (UᵀY, ||Y||², the TSQR R blocks) which every
  rank reduces in the same fixed order and then uses to take identical rank
  decisions redundantly.  `row_partition` and `reduce_partials_fixed_order`
  define that contract; tests/test_multiproc.py checks it with gloo at
  world_size 2 against the unsharded computation.
"""

from __future__ import annotations

import os


def dist_env():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) block of n units owned by `rank` (balanced, ordered)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def row_partition(n_rows: int, world: int) -> list[tuple[int, int]]:
    """Row slabs of every n_x-tall factor, one per rank (the GPU-level analogue of
    the per-CTA row ranges inside the persistent sweep kernel)."""
    return [shard_range(n_rows, r, world) for r in range(world)]


def max_over_ranks(value: float, group=None, device=None) -> float:
    """Job time = slowest rank (timing rule for multi-GPU numbers)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def reduce_partials_fixed_order(local, group=None):
    """Sum per-rank partial arrays so that EVERY rank obtains bit-identical
    results: gather all partials and add them in rank order (an all-reduce's
    internal order is not part of NCCL's contract, SURVEY §7 hard part 4)."""
    import torch
    import torch.distributed as dist

    t = torch.as_tensor(local, dtype=torch.float64)
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return t.clone()
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t.contiguous(), group=group)
    out = torch.zeros_like(t)
    for p in parts:
        out += p
    return out
