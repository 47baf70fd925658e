"""One IC Hessian apply at the C5 shape on ONE GPU (3-D convection-diffusion 256^3 = 16.8M dofs,
nu = 1/50, w = (1,1,1)/sqrt(3) + the rotating field in x-y, per-node upwind 7-point, 64^3 sensors,
sigma 0.005, prior (I+0.02L)^-1 per side, r_max 64) at a reduced number of time steps (the full
n_t = 4096 takes minutes per apply on the physical-space path; C5's 2/4/8-GPU sharding of that
path is not built).  usage: python tools/c5_probe.py [n_side] [n_t]"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1703_05638_b200 as lp

n_side = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n_t = int(sys.argv[2]) if len(sys.argv) > 2 else 16
grid = lp.build_grid(n_side, 3)
w0 = (3 ** -0.5,) * 3
K = lp.SpaceTimeOperator(lp.assemble_convdiff(grid, 1 / 50, w0, field="rotating"), lp.build_time_grid(n_t, T=n_t / 4096))
bn = 1.0 / (0.005 ** 2 * K.time.tau * grid.m_scale)
cov = lp.CovarianceSpec(bn, 1.0, 1.0, prior_delta=1.0, prior_gamma=0.02)
layout = lp.make_sensor_subgrid(grid, n_side // 4)
ctx = lp.HessianContext(mode="ic", operator=K, layout=layout, cov=cov, pol=lp.TruncationPolicy(1e-8, 64))
v = torch.as_tensor(np.random.default_rng(4).standard_normal(grid.n_x), device="cuda")
v /= v.norm()
for i in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = ctx.apply(v)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"C5 shape n_side {n_side} n_t {n_t} (tau = 1/4096): apply {1e3*(t1-t0):.1f} ms = "
          f"{1e3*(t1-t0)/(2*n_t):.1f} ms per time step, max rank {ctx.rank_trace[-1]}, "
          f"|out| {float(out.norm()):.4e}, launches {ctx._dev.launches()}, "
          f"mem {torch.cuda.max_memory_allocated()/2**30:.1f} GiB torch", flush=True)
