"""Time one convection-diffusion IC Hessian apply at the C3 size (nu = 1/20, 64x64
sensors, prior (I+0.05L)^-1 per side, r_max 48).
usage: python tools/c3_probe.py [n_side] [n_t] [rotating|const] [galerkin|upwind]
Default: C3 as specified — Galerkin Q1, rotating wind."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1703_05638_b200 as lp

n_side = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n_t = int(sys.argv[2]) if len(sys.argv) > 2 else 64
grid = lp.build_grid(n_side)
field = sys.argv[3] if len(sys.argv) > 3 else "rotating"
scheme = sys.argv[4] if len(sys.argv) > 4 else "galerkin"
K = lp.SpaceTimeOperator(lp.assemble_convdiff(grid, 0.05, (0.0, 0.0) if field == "rotating" else (1.0, -0.5),
                                              field=field, scheme=scheme), lp.build_time_grid(n_t))
bn = 1.0 / (0.01 ** 2 * K.time.tau * grid.m_scale)
cov = lp.CovarianceSpec(bn, 1.0, 1.0, prior_delta=1.0, prior_gamma=0.05)
layout = lp.make_sensor_subgrid(grid, min(64, n_side // 2))
ctx = lp.HessianContext(mode="ic", operator=K, layout=layout, cov=cov, pol=lp.TruncationPolicy(1e-8, 48))
v = torch.as_tensor(np.random.default_rng(2).standard_normal(grid.n_x), device="cuda")
v /= v.norm()
for i in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = ctx.apply(v)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"n_side {n_side} n_t {n_t}: apply {1e3*(t1-t0):.1f} ms, max rank {ctx.rank_trace[-1]}, "
          f"launches {ctx._dev.launches()}", flush=True)
