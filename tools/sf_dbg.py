import os, sys
import numpy as np
sys.path.insert(0, '.')
import paper_1703_05638_b200 as lp
from oracle import lrk_oracle as O
n_side, n_t = int(sys.argv[1]), int(sys.argv[2])
grid = lp.build_grid(n_side, 3)
K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(n_t))
rng = np.random.default_rng(1)
rhs = lp.LowRankMat(rng.standard_normal((grid.n_x, 1)), np.eye(n_t)[:, :1])
pol = lp.TruncationPolicy(1e-8, 64)
for form in ("0", "1"):
    os.environ["LRK_SFLUSH"] = form
    os.environ["LRK_SF_DEBUG"] = os.environ.get("DBG", "0") if form == "1" else "0"
    tr = []
    Y = lp.st_solve_sweep(K, rhs, pol, trace=tr)
    print(form, tr, np.linalg.svd(lp.lr_to_dense(Y), compute_uv=False)[:6], flush=True)
