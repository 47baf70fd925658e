"""Full-size C4 apply with the n_x-sharded streaming sweep driven on ONE device (all shards'
kernels launched by one process, same exchange protocol) against the unsharded apply."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1703_05638_b200 as lp
from paper_1703_05638_b200 import _lib

def make():
    grid = lp.build_grid(128, 3)
    K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(2048))
    bn = 1.0 / (0.005 ** 2 * K.time.tau * grid.m_scale)
    cov = lp.CovarianceSpec(bn, 1.0, 1.0, prior_delta=1.0, prior_gamma=0.02)
    layout = lp.make_sensor_subgrid(grid, 32, time_every=4)
    return grid, lp.HessianContext(mode="ic", operator=K, layout=layout, cov=cov, pol=lp.TruncationPolicy(1e-8, 64))

grid, ctx = make()
v = torch.as_tensor(np.random.default_rng(5).standard_normal(grid.n_x), device="cuda"); v /= v.norm()
ref = ctx.apply(v).clone(); r0 = ctx.rank_trace[-1]
fw0, ob0, bw0 = ctx.last_traces()
for shards in (2, 4, 8):
    g2, c2 = make()
    assert _lib.get_lib().lrk_set_emulated_shards(c2._dev.handle, shards) == 0
    c2.apply(v)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = c2.apply(v)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    fw, ob, bw = c2.last_traces()
    rel = float((out - ref).norm() / ref.norm())
    print(f"C4 full size, {shards} shards on one device: rel diff vs unsharded {rel:.2e}, rank traces equal {fw == fw0 and bw == bw0 and ob == ob0}, max rank {c2.rank_trace[-1]} ({r0}), {1e3*dt:.0f} ms (serialised shards)")
