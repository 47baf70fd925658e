"""FP64 tensor-pipe reference numbers on this GPU: cuBLAS DGEMM (torch fp64
matmul) vs our DMMA DST (lrk_step_solve on the heat operator = 4 DST GEMM
passes + one scaling)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1703_05638_b200 as lp

def bench(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

for n in (4096, 8192):
    A = torch.randn(n, n, dtype=torch.float64, device="cuda"); B = torch.randn(n, n, dtype=torch.float64, device="cuda")
    ms = bench(lambda: A @ B, 5)
    print(f"cuBLAS DGEMM {n}^3: {2*n**3/ms/1e9:.1f} TF/s")
A = torch.randn(64, 512, 512, dtype=torch.float64, device="cuda"); B = torch.randn(512, 512, dtype=torch.float64, device="cuda")
ms = bench(lambda: A @ B)
print(f"cuBLAS batched 64x512^3: {64*2*512**3/ms/1e9:.1f} TF/s")
for n_side, nc in ((512, 1), (512, 16), (256, 64), (128, 64)):
    grid = lp.build_grid(n_side)
    K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(8))
    X = torch.randn(nc, grid.n_x, dtype=torch.float64, device="cuda").T
    ms = bench(lambda: K.solve_step(X))
    fl = 4 * 2 * n_side**3 * nc
    print(f"lrk DST step solve n_side {n_side} x {nc} cols: {ms*1e3:.1f} us, {fl/ms/1e9:.1f} TF/s")
