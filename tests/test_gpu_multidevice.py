"""The n_x-sharded Hessian apply across real GPUs (one process per GPU, NCCL
for the handle exchange, peer-memory exchange inside the sweeps): every rank
must return the unsharded result with identical rank traces.  Needs >= 2 GPUs
on the node and skips otherwise (the single-GPU tiers cover the same kernels
and protocol through tests/test_gpu_config_scale.py::test_nx_sharded_*)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _make(lp):
    n_side, n_t = 48, 32
    grid = lp.build_grid(n_side, 3)
    K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(n_t))
    bn = 1.0 / (0.005 ** 2 * K.time.tau * grid.m_scale)
    cov = lp.CovarianceSpec(bn, 1.0, 1.0, prior_delta=1.0, prior_gamma=0.02)
    layout = lp.make_sensor_subgrid(grid, 12, time_every=4)
    ctx = lp.HessianContext(mode="ic", operator=K, layout=layout, cov=cov,
                            pol=lp.TruncationPolicy(1e-8, 64))
    v = np.random.default_rng(3).standard_normal(grid.n_x)
    return ctx, v / np.linalg.norm(v)


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_1703_05638_b200 as lp

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        ctx, v = _make(lp)
        ref = ctx.apply(v)
        tr_ref = ctx.last_traces()
        assert ctx.shard() == (rank, world)
        out = ctx.apply(v)
        tr = ctx.last_traces()
        out2 = ctx.apply(v)          # a second apply reuses the exchange slots
        q.put((rank, float(np.abs(out - ref).max() / np.abs(ref).max()), tr == tr_ref,
               float(np.abs(out2 - out).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs on the node")
@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_apply_across_gpus_matches_unsharded(world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp

    port = _free_port()
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    procs = [mpc.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, err, same_trace, drift in res:
        assert err <= 1e-11, (rank, err)
        assert same_trace, rank
        assert drift == 0.0, (rank, drift)
