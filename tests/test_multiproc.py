"""N>1 host logic with torch.distributed (gloo, world_size 2, CPU).

1. probe sharding: every probe applied exactly once, job time = max over ranks;
2. spectral-row sharding of a sweep flush: each rank holds a row slab of the
   n_x-tall factors, partial sums are reduced in a fixed order, and every rank
   takes the SAME rank decision and obtains the same truncated pane as the
   unsharded computation (the contract the multi-GPU sweep relies on).
The numpy flush model below mirrors the device algorithm (block CGS2 against
the orthonormal pane + QR of the remainder + SVD of the Brand core); the
oracle supplies _rank_cut.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import lrk_oracle as O
from paper_1703_05638_b200 import parallel as par


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _flush_sharded(U, sig, Y, rows, reduce):
    """One Brand flush with U, Y row-sharded: partials -> reduce -> redundant core SVD."""
    lo, hi = rows
    Ul, Yl = U[lo:hi], Y[lo:hi]
    C1 = reduce(Ul.T @ Yl)
    P = Yl - Ul @ C1
    C2 = reduce(Ul.T @ P)
    P = P - Ul @ C2
    # remainder QR via the Gram of the (already twice-projected) remainder is
    # what a TSQR reduces; here the R of the stacked local QRs
    Rl = np.linalg.qr(P, mode="r") if P.shape[0] else np.zeros((0, Y.shape[1]))
    Rl = np.vstack([Rl, np.zeros((Y.shape[1] - Rl.shape[0], Y.shape[1]))]) if Rl.shape[0] < Y.shape[1] else Rl
    Rs = reduce_stack(Rl)
    Rp = np.linalg.qr(Rs, mode="r")
    r, p = U.shape[1], Y.shape[1]
    core = np.zeros((r + p, r + p))
    core[:r, :r] = np.diag(sig)
    core[:r, r:] = C1 + C2
    core[r:, r:] = Rp
    s = np.linalg.svd(core, compute_uv=False)
    return O.rank_cut(s, 1e-8), s


reduce_stack = None


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1. probe sharding
        n_probe = 7
        lo, hi = par.shard_range(n_probe, rank, world)
        mine = list(range(lo, hi))
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        t_job = par.max_over_ranks(0.1 * (rank + 1))
        # 2. spectral-row sharded flush
        rng = np.random.default_rng(0)
        n_x, r, p = 101, 6, 4
        U = np.linalg.qr(rng.standard_normal((n_x, r)))[0]
        sig = np.logspace(0, -6, r)
        Y = U @ rng.standard_normal((r, p)) * 0.3 + 1e-9 * rng.standard_normal((n_x, p))
        rows = par.row_partition(n_x, world)[rank]

        def reduce(x):
            return par.reduce_partials_fixed_order(x).numpy()

        global reduce_stack

        def _stack(Rl):
            t = torch.as_tensor(Rl)
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t.contiguous())
            return np.vstack([x.numpy() for x in parts])

        reduce_stack = _stack
        rk, s = _flush_sharded(U, sig, Y, rows, reduce)
        decisions = [None] * world
        dist.all_gather_object(decisions, (rk, s.tobytes()))
        q.put((rank, allp, t_job, decisions, rk, s))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding_and_flush_determinism():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort()
    # every probe exactly once, in rank order
    allp = res[0][1]
    assert sorted(x for part in allp for x in part) == list(range(7))
    assert res[0][2] == res[1][2] == pytest.approx(0.2)
    # identical rank decisions and bit-identical singular values on both ranks
    d0, d1 = res[0][3], res[1][3]
    assert d0 == d1
    # ... equal to the unsharded flush
    rng = np.random.default_rng(0)
    n_x, r, p = 101, 6, 4
    U = np.linalg.qr(rng.standard_normal((n_x, r)))[0]
    sig = np.logspace(0, -6, r)
    Y = U @ rng.standard_normal((r, p)) * 0.3 + 1e-9 * rng.standard_normal((n_x, p))
    W1 = np.hstack([U * sig, Y])
    s_ref = np.linalg.svd(W1, compute_uv=False)
    assert res[0][4] == O.rank_cut(s_ref, 1e-8)
    np.testing.assert_allclose(res[0][5][: res[0][4]], s_ref[: res[0][4]], rtol=1e-12)


def test_shard_range_partitions():
    for n in (0, 1, 5, 148, 65536):
        for w in (1, 2, 3, 8):
            rs = [par.shard_range(n, k, w) for k in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1


def _handle_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = bytes((17 * rank + i) % 256 for i in range(par.IPC_HANDLE_BYTES))
        got = par.exchange_handles(mine)
        # a failure on ONE rank is seen by every rank (no rank left in a collective)
        assert par._all_ranks_ok(True) is True
        assert par._all_ranks_ok(rank != 1) is False
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


def test_ipc_handle_exchange_is_rank_ordered():
    """The setup step of the n_x-sharded sweeps: every rank's 64-byte CUDA IPC
    handle (lrk_shard_setup) reaches every rank, concatenated in rank order,
    which is what lrk_shard_connect indexes by peer rank."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_handle_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    want = b"".join(bytes((17 * r + i) % 256 for i in range(par.IPC_HANDLE_BYTES))
                    for r in range(world))
    assert res[0][1] == want and res[1][1] == want


def test_shard_context_is_a_noop_without_a_process_group():
    class _Ctx:
        handle = None

    assert par.shard_context(_Ctx()) == (0, 1)
