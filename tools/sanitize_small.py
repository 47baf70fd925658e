"""Small Hessian applies for compute-sanitizer (memcheck / racecheck / synccheck).

Covers, at sizes the sanitizer finishes in a minute: the persistent sweep
kernel (resident rows, split arrive/wait grid barriers), the streaming-flush
sweep (cp.async rings, last-CTA tickets) unsharded and as 2 emulated n_x
shards (peer-slot exchange, release/acquire flags, tail kernels), the
truncation kernel, the DMMA GEMMs and the Gram kernels (lr_dot).
Usage: compute-sanitizer --tool <tool> python tools/sanitize_small.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1703_05638_b200 as lp  # noqa: E402
from paper_1703_05638_b200 import _lib  # noqa: E402


def one(n_side, dim, n_t, sensors, every, form, shards):
    os.environ.pop("LRK_SFLUSH", None)
    if form is not None:
        os.environ["LRK_SFLUSH"] = form
    grid = lp.build_grid(n_side, dim)
    K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(n_t))
    bn = 1.0 / (0.01 ** 2 * K.time.tau * grid.m_scale)
    cov = lp.CovarianceSpec(bn, 1.0, 1.0, prior_delta=1.0, prior_gamma=0.05)
    ctx = lp.HessianContext(mode="ic", operator=K,
                            layout=lp.make_sensor_subgrid(grid, sensors, time_every=every),
                            cov=cov, pol=lp.TruncationPolicy(1e-8, 32))
    if shards > 1:
        assert _lib.get_lib().lrk_set_emulated_shards(ctx._dev.handle, shards) == 0
    v = np.random.default_rng(0).standard_normal(grid.n_x)
    out = ctx.apply(v / np.linalg.norm(v))
    print(f"n_side {n_side} d {dim} n_t {n_t} form {form} shards {shards}: |out| "
          f"{np.linalg.norm(out):.6e} rank {ctx.rank_trace[-1]}", flush=True)
    return out


a = one(16, 2, 12, 4, 1, "0", 1)       # persistent kernel
b = one(16, 2, 12, 4, 1, "1", 1)       # streaming flush
c = one(16, 2, 12, 4, 1, "1", 2)       # streaming flush, 2 emulated shards
assert np.allclose(a, b, rtol=0, atol=1e-10 * np.abs(a).max())
assert np.allclose(b, c, rtol=0, atol=1e-10 * np.abs(a).max())
one(8, 3, 8, 4, 2, "1", 1)             # 3-D, time-subsampled sensors
A = lp.lr_from_dense(np.random.default_rng(1).standard_normal((60, 9)) @
                     np.random.default_rng(2).standard_normal((9, 14)), lp.TruncationPolicy(1e-10))
print("lr_dot", lp.lr_dot(A, A), "rank", A.r)
