"""HBM roofline of the streaming kernels at config scale (GPU box).

Times, with CUDA events on the launch stream after warm-up, the two
bandwidth-bound entry points the north star names outside the sweep:
  * K.apply on a rank-r field (the stencil SpMM S W1 plus -M W1),
    algorithmic bytes 8 n_x r (read W1) + 16 n_x r (write the two blocks);
  * lr_dot of two rank-r fields (the Gram products over n_x and n_t),
    algorithmic bytes 8 (n_x + n_t)(r_a + r_b).
Prints one JSON line per case with achieved GB/s against MEASURED_PEAKS.json.
Usage: python tools/hbm_roofline.py [--n-side 128] [--d 3] [--r 64]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1703_05638_b200 as lp  # noqa: E402


def peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 7700.0, "fallback"


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def field(n_x, n_t, r, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    W1 = torch.randn(r, n_x, device="cuda", dtype=torch.float64, generator=g).t()
    W2 = torch.randn(r, n_t, device="cuda", dtype=torch.float64, generator=g).t()
    return lp.LowRankMat(W1, W2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-side", type=int, default=128)
    ap.add_argument("--d", type=int, default=3)
    ap.add_argument("--n-t", type=int, default=2048)
    ap.add_argument("--r", type=int, default=64)
    args = ap.parse_args()
    peak, kind = peak_gbs()
    grid = lp.build_grid(args.n_side, args.d)
    K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(args.n_t))
    n_x, n_t, r = grid.n_x, args.n_t, args.r
    A = field(n_x, n_t, r, 1)
    B = field(n_x, n_t, r, 2)
    cases = [
        ("K.apply (stencil SpMM + mass)", lambda: K.apply(A), 8.0 * n_x * r + 16.0 * n_x * r + 24.0 * n_t * r),
        ("lr_dot (Gram over n_x and n_t)", lambda: lp.lr_dot(A, B), 8.0 * (n_x + n_t) * 2 * r),
    ]
    for name, fn, nbytes in cases:
        t = timed(fn)
        gbs = nbytes / t / 1e9
        print(json.dumps({"kernel": name, "n_x": n_x, "n_t": n_t, "r": r, "ms": t * 1e3,
                          "alg_bytes": nbytes, "achieved_gbs": gbs, "peak_gbs": peak,
                          "peak_kind": kind, "frac": gbs / peak}))


if __name__ == "__main__":
    main()
