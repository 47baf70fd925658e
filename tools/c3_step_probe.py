"""Wall vs device time of the convection-diffusion step solve at C3 size
(one column, the preconditioned Richardson path): launch-bound or GPU-bound?"""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_1703_05638_b200 as lp

n_side = int(sys.argv[1]) if len(sys.argv) > 1 else 512
grid = lp.build_grid(n_side)
K = lp.SpaceTimeOperator(lp.assemble_convdiff(grid, 0.05, (0.0, 0.0), field="rotating"), lp.build_time_grid(1024))
B = torch.randn(grid.n_x, 1, device="cuda", dtype=torch.float64)
for _ in range(3):
    K.solve_step(B)
torch.cuda.synchronize()
reps = 50
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); e0.record()
for _ in range(reps):
    K.solve_step(B)
e1.record(); t1 = time.perf_counter()
torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"step solve: host issue {1e3*(t1-t0)/reps:.3f} ms/solve, device {e0.elapsed_time(e1)/reps:.3f} ms/solve, wall {1e3*(t2-t0)/reps:.3f} ms/solve")
