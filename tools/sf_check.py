"""Streaming-flush sweep vs the persistent kernel on the same apply (debug aid).
usage: python tools/sf_check.py n_side dim n_t [r_max]"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1703_05638_b200 as lp

n_side, dim, n_t = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rmax = int(sys.argv[4]) if len(sys.argv) > 4 else 64
grid = lp.build_grid(n_side, dim)
K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(n_t))
bn = 1.0 / (0.005 ** 2 * K.time.tau * grid.m_scale)
cov = lp.CovarianceSpec(bn, 1.0, 1.0, prior_delta=1.0, prior_gamma=0.02)
layout = lp.make_sensor_subgrid(grid, max(n_side // 4, 1), time_every=4)
v = np.random.default_rng(3).standard_normal(grid.n_x)
v /= np.linalg.norm(v)
res = {}
for form in ("0", "1"):
    os.environ["LRK_SFLUSH"] = form
    ctx = lp.HessianContext(mode="ic", operator=K, layout=layout, cov=cov,
                            pol=lp.TruncationPolicy(1e-8, rmax))
    out = ctx.apply(v)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = ctx.apply(v)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    res[form] = (out, ctx.last_traces(), dt)
    fw, ob, bw = ctx.last_traces()
    print(f"LRK_SFLUSH={form}: {1e3*dt:.1f} ms, |out| {np.linalg.norm(out):.6e}, fwd {fw[:12]}.. obs {ob} bwd {bw[:12]}..")
a, b = res["0"][0], res["1"][0]
print("rel diff", np.linalg.norm(a - b) / np.linalg.norm(a), "traces equal", res["0"][1] == res["1"][1])
