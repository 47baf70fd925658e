"""Multi-GPU host logic: one process per GPU, torch.distributed for plumbing.

`shard_context` turns the sweeps of a device context into n_x-sharded sweeps
across the ranks of a process group: each rank keeps the whole
operator and replicated n_x inputs/outputs, runs the forward and adjoint
sweeps on its own row slab, and exchanges the small per-pass rank totals
through peer-mapped memory inside the kernels (include/lrk.h, lrk_shard_*);
torch.distributed only carries the 64-byte CUDA IPC handles at setup.

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


IPC_HANDLE_BYTES = 64


def exchange_handles(mine: bytes, group=None, device=None) -> bytes:
    """All-gather one fixed-size byte string per rank, in rank order (the CUDA
    IPC handles of lrk_shard_setup).  Works on any backend: the payload rides
    in a uint8 tensor on `device` (CPU for gloo, the rank's GPU for nccl)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if device is None:
        device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor(list(mine), dtype=torch.uint8, device=device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    return b"".join(bytes(p.cpu().tolist()) for p in parts)


def _all_ranks_ok(ok: bool, group=None, device=None) -> bool:
    """True when `ok` holds on every rank (one small MIN all-reduce): every
    rank learns about a failure anywhere, so nobody is left waiting in the
    next collective."""
    import torch
    import torch.distributed as dist

    if device is None:
        device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([1.0 if ok else 0.0], device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return bool(t.item() == 1.0)


def shard_context(dev_ctx, group=None, device=None) -> tuple[int, int]:
    """Shard the sweeps of `dev_ctx` (a _lib.Context with its operator
    installed) by n_x rows across the ranks of `group`.  Returns (rank, world).
    With a world of one this is a no-op.  Collective: every rank must call it;
    a failure on any rank raises RuntimeError on all of them."""
    import ctypes

    import torch.distributed as dist

    from . import _lib

    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if world == 1:
        return 0, 1
    lib = _lib.get_lib()
    h = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    st = lib.lrk_shard_setup(dev_ctx.handle, rank, world, h)
    msg = lib.lrk_last_error(dev_ctx.handle).decode() if st else ""
    if not _all_ranks_ok(st == 0, group, device):
        raise RuntimeError(f"lrk_shard_setup failed on a rank (here: status {st} {msg})")
    handles = exchange_handles(h.raw, group=group, device=device)
    buf = ctypes.create_string_buffer(handles, len(handles))
    st = lib.lrk_shard_connect(dev_ctx.handle, buf)
    msg = lib.lrk_last_error(dev_ctx.handle).decode() if st else ""
    if not _all_ranks_ok(st == 0, group, device):
        raise RuntimeError(f"lrk_shard_connect failed on a rank (here: status {st} {msg})")
    return rank, world
