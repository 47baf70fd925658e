"""Eigen run at a BASELINE configuration on the GPU: lr_arnoldi with the
config's m_a around HessianContext.apply, Ritz pairs, posterior variance with
the config prior.  Prints one JSON line (kept under profiles/): iterations,
matvecs/s over the run's own Arnoldi basis (m_a / sum of apply
times), wall time of the whole run, leading Ritz values, basis orthogonality,
a symmetry probe <u, H v> = <H u, v>, variance range.

usage: python tools/config_arnoldi.py C2|C3|C4 [m_a] [fixed|stop]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1703_05638_b200 as lp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
default_ma = {"C2": 50, "C3": 64, "C4": 100}[name]
m_a = int(sys.argv[2]) if len(sys.argv) > 2 else default_ma
mode = sys.argv[3] if len(sys.argv) > 3 else "fixed"

if name == "C3":
    n_side, n_t, seed = 512, 1024, 2
    grid = lp.build_grid(n_side)
    K = lp.SpaceTimeOperator(lp.assemble_convdiff(grid, 1 / 20, (0.0, 0.0), field="rotating",
                                                  scheme="galerkin"), lp.build_time_grid(n_t))
    bn = 1.0 / (0.01 ** 2 * K.time.tau * grid.m_scale)
    cov = lp.CovarianceSpec(bn, 1.0, 1.0, prior_delta=1.0, prior_gamma=0.05)
    ctx = lp.HessianContext(mode="ic", operator=K, layout=lp.make_sensor_subgrid(grid, 64), cov=cov,
                            pol=lp.TruncationPolicy(1e-8, 48))
else:
    cfg = bench.CONFIGS[name]
    seed = cfg["seed"]
    ctx, grid = bench.make_context(cfg, lp)

v1 = torch.as_tensor(lp.start_vector(grid.n_x, start="random", seed=seed), device="cuda")
times = []


def apply(v):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = ctx.apply(v)
    torch.cuda.synchronize()
    times.append(time.perf_counter() - t0)
    return out


stop = lp.StopRule(m_a=m_a, eps_eig=1e-1, check_every=(m_a + 1 if mode == "fixed" else 10))
t0 = time.perf_counter()
res = lp.lr_arnoldi(apply, v1, ctx.pol, stop, rank_source=ctx.rank_trace)
t_arn = time.perf_counter() - t0
n_apply = len(times)
summ = lp.build_summary(res.ritz_values, res.ritz_vectors, 1.0, 1e-1, prior=ctx.prior)
torch.cuda.synchronize()
t_all = time.perf_counter() - t0
# symmetry probe with two seeded vectors (not part of the timing)
rng = np.random.default_rng(seed + 100)
u = torch.as_tensor(rng.standard_normal(grid.n_x), device="cuda")
w = torch.as_tensor(rng.standard_normal(grid.n_x), device="cuda")
u, w = u / u.norm(), w / w.norm()
Hu, Hw = ctx.apply(u), ctx.apply(w)
sym = float(abs((u @ Hw) - (Hu @ w)) / max(abs(float(u @ Hw)), 1e-300))
ritz = np.sort(res.ritz_values.real)[::-1]
H = res.H
print(json.dumps({
    "config": name, "m_a": m_a, "stop": mode, "iterations": res.iterations, "applies": n_apply,
    "matvecs_per_s_over_the_arnoldi_basis": n_apply / sum(times),
    "mean_apply_ms": 1e3 * sum(times) / n_apply,
    "arnoldi_wall_s": t_arn, "with_ritz_vectors_and_variance_s": t_all,
    "orthogonalisation_and_host_share": 1.0 - sum(times) / t_arn,
    "max_rank": int(max(res.rank_trace)), "breakdown": bool(res.breakdown),
    "ritz_leading": [float(x) for x in ritz[:12]],
    "ritz_retained_ge_0.1": int((ritz >= 1e-1).sum()),
    "ritz_max_imag": float(np.abs(res.ritz_values.imag).max()),
    "hessenberg_asymmetry": float(np.abs(H[:-1] - H[:-1].T).max() / np.abs(H).max()),
    "basis_gram_defect": res.gram_defect(),
    "symmetry_probe_rel": sym,
    "variance_min": float(summ.variance_field.min()), "variance_max": float(summ.variance_field.max()),
    "prior_variance_max": float(ctx.prior.diag(2).max()),
}))
