"""Time one C4-shaped IC Hessian apply (3-D 7-point heat, n_side 128, 32^3 sensors
every 4th step, prior (I+0.02L)^-1 per side, sigma 0.005, r_max 64) at a given n_t."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1703_05638_b200 as lp

n_side = int(sys.argv[1]) if len(sys.argv) > 1 else 128
n_t = int(sys.argv[2]) if len(sys.argv) > 2 else 64
grid = lp.build_grid(n_side, 3)
K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(n_t))
bn = 1.0 / (0.005 ** 2 * K.time.tau * grid.m_scale)
cov = lp.CovarianceSpec(bn, 1.0, 1.0, prior_delta=1.0, prior_gamma=0.02)
layout = lp.make_sensor_subgrid(grid, n_side // 4, time_every=4)
ctx = lp.HessianContext(mode="ic", operator=K, layout=layout, cov=cov, pol=lp.TruncationPolicy(1e-8, 64))
v = torch.as_tensor(np.random.default_rng(3).standard_normal(grid.n_x), device="cuda")
v /= v.norm()
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
for i in range(reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = ctx.apply(v)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"n_side {n_side} n_t {n_t}: apply {1e3*(t1-t0):.1f} ms, max rank {ctx.rank_trace[-1]}, |out| {float(out.norm()):.4e}")
