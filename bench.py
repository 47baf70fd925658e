#!/usr/bin/env python
"""Benchmark: low-rank space-time Hessian matvecs/s on the C2 workload.

Workload (BASELINE.json configs[1], the metric's config): 2-D heat equation on
[0,1]^2, 256x256 interior grid (n_x = 65,536), n_t = 512, T = 1, implicit
Euler, fp64; initial-condition parameter; 32x32 uniform point-sensor subgrid
observed at every step; noise sigma = 0.01 (pointwise weight 1/sigma^2,
SURVEY Appendix D1); prior (delta I + gamma L)^-2 with delta = 1, gamma = 0.05
(square root applied on both sides); truncation eps0 =
1e-8, rank cap 32; seed 1.  Operator: Q1 bilinear FEM stiffness with lumped
mass (9-point stencil), exactly the config's discretisation.

One step = one prior-preconditioned misfit Hessian apply (forward sweep, obs,
adjoint sweep; hessian.py:211-226) on a seeded N(0,1) unit probe already
resident in HBM.  L2 is flushed (512 MiB write) before every timed step.
Multi-GPU: every rank applies H~ to its own probes (independent units, no
data-path collective) -> weak scaling; time = max over ranks.

--impl reference times the reference algorithm on the host CPU (oracle/
restatement, SuperLU + LAPACK, validated against the reference in
tests/test_oracle_golden.py), all host cores as independent processes, each
step a bounded prefix sample of the same apply (see _cpu_sample).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_SIDE, N_T, SENSORS, SIGMA, EPS0, R_MAX, SEED, P_FLUSH = 256, 512, 32, 0.01, 1e-8, 32, 1, 4
PRIOR_DELTA, PRIOR_GAMMA = 1.0, 0.05
STENCIL = "q1"
CPU_SAMPLE_STEPS = 32   # time steps per sweep in one CPU sample (of 512)
L2_FLUSH_BYTES = 512 << 20

WORKLOAD = ("C2: 2D heat 256x256 (n_x=65536), n_t=512, Q1 FEM (lumped mass, 9-point), IC "
            "parameter, 32x32 point sensors every step, sigma=0.01 (w=1/sigma^2), prior "
            "(I+0.05L)^-2, eps0=1e-8, r_max=32, compress_every=4, seed 1")


def problem_scalars():
    h = 1.0 / (N_SIDE + 1)
    tau = 1.0 / N_T
    beta_noise = 1.0 / (SIGMA ** 2 * tau * h * h)  # w = beta_noise*tau*h^2 = 1/sigma^2
    beta_prior = 1.0 / (h * h)  # unused by the apply; gamma_prior = 1 scales nothing
    return h, tau, beta_noise, beta_prior


def sensor_mask():
    stride = N_SIDE // SENSORS
    idx = stride // 2 + stride * np.arange(SENSORS)
    mask = np.zeros(N_SIDE * N_SIDE, bool)
    mask[(idx[:, None] * N_SIDE + idx[None, :]).ravel()] = True
    return mask


def probes(n, count, seed):
    rng = np.random.default_rng(seed)
    V = rng.standard_normal((n, count))
    return V / np.linalg.norm(V, axis=0)


# ------------------------------------------------------------------ CPU arm
def _cpu_sample(args):
    """One bounded sample of the reference apply: the C2 operator (same n_x,
    tau = 1/512, sensors, weights) swept over CPU_SAMPLE_STEPS of the 512 time
    steps in each direction.  Returns seconds; the matvec rate is extrapolated
    linearly in n_t (cost per step is ~constant once the rank settles)."""
    seed, reps = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import lrk_oracle as O

    h, tau, bn, bp = problem_scalars()
    P = O.Problem(N_SIDE, CPU_SAMPLE_STEPS, sensor_mask(), bn, 1.0, EPS0, R_MAX,
                  T=CPU_SAMPLE_STEPS * tau, stencil=STENCIL, prior=(PRIOR_DELTA, PRIOR_GAMMA))
    v = probes(N_SIDE * N_SIDE, 1, seed)[:, 0]
    t0 = time.perf_counter()
    for _ in range(reps):
        O.hessian_ic(P, v)
    return (time.perf_counter() - t0) / reps


def cpu_arm(steps: int, warmup: int, reps: int = 1):
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores, initializer=_limit_threads) as pool:
        for _ in range(warmup):
            pool.map(_cpu_sample, [(SEED + i, 1) for i in range(cores)])
        t0 = time.perf_counter()
        per = []
        for _ in range(steps):
            per += pool.map(_cpu_sample, [(SEED + i, reps) for i in range(cores)])
        wall = time.perf_counter() - t0
    frac = CPU_SAMPLE_STEPS / N_T
    # aggregate: cores x steps x reps samples, each frac of a matvec
    value = cores * steps * reps * frac / wall
    return value, cores, float(np.median(per)), wall


def _limit_threads():
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"


# ------------------------------------------------------------------ helpers
class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    polled every 5 ms from a background thread (initialised before the region
    starts, so its setup is outside it); nvidia-smi -lms 200 if NVML is
    unavailable."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits (nvml.h)
    BITS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
            ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = None
        self.samples = []
        try:
            import threading
            import pynvml
            pynvml.nvmlInit()
            h = None
            try:
                import torch
                pr = torch.cuda.get_device_properties(index)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.nvml, self.h = pynvml, h
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
        except Exception:
            self.nvml = None

    def _poll(self):
        nv, h = self.nvml, self.h
        while not self.stop.is_set():
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                self.samples.append((sm, rs))
            except Exception:
                pass
            self.stop.wait(0.005)

    def __enter__(self):
        if self.nvml is not None:
            self.thread.start()
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.nvml is not None:
            self.stop.set()
            self.thread.join(timeout=2)
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        if self.nvml is not None:
            sm = [v for v, _ in self.samples]
            reasons = {name for name, bit in self.BITS for _, r in self.samples if r & bit}
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.mx,
                    "reasons": sorted(reasons), "samples": len(sm), "source": "nvml 5 ms"}
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            parts = [p.strip() for p in l.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except (ValueError, IndexError):
                continue
            for name, val in zip(names, parts[2:]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi -lms 200"}


def measured_hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    """Per-launch DRAM bytes of the sweep kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_sweep_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch"), d.get("source")
    except Exception:
        return None, None


# ------------------------------------------------------------------ GPU arm
def gpu_arm(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1703_05638_b200 as lp
    from paper_1703_05638_b200 import _lib
    from ctypes import byref, c_double, c_int64

    torch.cuda.set_device(local_rank)
    h, tau, bn, bp = problem_scalars()
    grid = lp.build_grid(N_SIDE)
    K = lp.SpaceTimeOperator(lp.assemble_heat(grid, STENCIL), lp.build_time_grid(N_T))
    cov = lp.CovarianceSpec(beta_noise=bn, beta_prior=bp, gamma_prior=1.0,
                            prior_delta=PRIOR_DELTA, prior_gamma=PRIOR_GAMMA)
    ctx = lp.HessianContext(mode="ic", operator=K, layout=lp.SensorLayout((), sensor_mask()),
                            cov=cov, pol=lp.TruncationPolicy(EPS0, R_MAX), compress_every=P_FLUSH)
    nprobe = args.steps + args.warmup
    V = probes(grid.n_x, nprobe, SEED * 1000 + rank)
    Vd = torch.as_tensor(V, device="cuda").T.contiguous()  # resident in HBM
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    lib = _lib.get_lib()
    h_dev = ctx._dev.handle

    for i in range(args.warmup):
        ctx.apply(Vd[i])
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    # ---------------- device-resident timed region
    lib.lrk_profile_enable(h_dev, 1)
    lib.lrk_profile_read(h_dev, None, None, None, 1)
    launches0 = ctx._dev.launches()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    ranks = []
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record()
            ctx.apply(Vd[args.warmup + i])
            evs[i][1].record()
            ranks.append(ctx.rank_trace[-1])
        torch.cuda.synchronize()
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = float(sum(step_ms))
    launches = ctx._dev.launches() - launches0
    sw_ms, sw_n, sw_bytes = c_double(0), c_int64(0), c_double(0)
    lib.lrk_profile_read(h_dev, byref(sw_ms), byref(sw_n), byref(sw_bytes), 1)
    lib.lrk_profile_enable(h_dev, 0)

    # ---------------- end-to-end through the public API with host buffers
    vh = torch.empty(grid.n_x, dtype=torch.float64).pin_memory()
    oh = torch.empty(grid.n_x, dtype=torch.float64).pin_memory()
    e2e_ev = []
    barrier()
    torch.cuda.synchronize()
    t_e2e = time.perf_counter()
    for i in range(args.steps):
        vh.copy_(torch.from_numpy(V[:, args.warmup + i]))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = ctx.apply(vh.to("cuda", non_blocking=True))
        oh.copy_(out, non_blocking=True)
        b.record()
        e2e_ev.append((a, b))
    torch.cuda.synchronize()
    t_e2e = time.perf_counter() - t_e2e
    barrier()
    e2e_ms = float(sum(a.elapsed_time(b) for a, b in e2e_ev))

    # max over ranks
    stats = torch.tensor([total_ms, e2e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
    total_ms, e2e_ms = float(stats[0]), float(stats[1])
    return {
        "total_ms": total_ms, "e2e_ms": e2e_ms, "launches": launches, "ranks": ranks,
        "sweep_ms": sw_ms.value, "sweep_n": sw_n.value, "sweep_bytes": sw_bytes.value,
        "clocks": clk.summary(), "n_x": grid.n_x, "e2e_wall_s": t_e2e,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = {"workload": WORKLOAD, "n_x": N_SIDE * N_SIDE, "n_t": N_T, "rank_cap": R_MAX,
           "eps0": EPS0, "parallelism": f"independent probes x{args.gpus} (replicas)",
           "l2": "flushed before every timed step (512 MiB write)",
           "solver_backend": "sweep (forward.py:133-188), DST-I eigenbasis"}

    if args.impl == "reference":
        if rank != 0:
            return
        value, cores, med, wall = cpu_arm(args.steps, args.warmup)
        sample = (f"per step: {cores} processes x 1 apply on the C2 operator over "
                  f"{CPU_SAMPLE_STEPS}/{N_T} time steps per sweep (extrapolated linearly in n_t); "
                  f"median sample {med:.2f}s")
        line = {"metric": "low-rank space-time Hessian matvecs/s", "value": value,
                "unit": "matvec/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded N(0,1) unit probes)", "config": cfg,
                "impl": "reference",
                "cpu_baseline": {"value": value, "unit": "matvec/s", "cores": cores,
                                 "kind": "port", "sample": sample},
                "e2e": {"value": value, "unit": "matvec/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = gpu_arm(args, rank, world, local_rank)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        value, cores, med, wall = cpu_arm(1, 0)
        cpu = {"value": value, "unit": "matvec/s", "cores": cores, "kind": "port",
               "sample": f"{cores} processes x 1 reference apply over {CPU_SAMPLE_STEPS}/{N_T} "
                         f"steps per sweep of the C2 operator (extrapolated in n_t); "
                         f"median sample {med:.2f}s"}
    if rank == 0:
        peak, peak_kind = measured_hbm_peak()
        per_launch_ms = res["sweep_ms"] / max(res["sweep_n"], 1)
        per_launch_bytes = res["sweep_bytes"] / max(res["sweep_n"], 1)
        achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9 if per_launch_ms > 0 else 0.0
        traffic, _src = ncu_traffic()
        n = args.gpus
        value = n * args.steps / (res["total_ms"] * 1e-3)
        line = {
            "metric": "low-rank space-time Hessian matvecs/s", "value": value, "unit": "matvec/s",
            "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res["total_ms"] / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded N(0,1) unit probes; no dataset)", "config": cfg,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "lrk::sweep_kernel", "peak_kind": peak_kind,
                         "alg_bytes_per_launch": per_launch_bytes,
                         "ms_per_launch": per_launch_ms},
            "cpu_baseline": cpu,
            "e2e": {"value": n * args.steps / (res["e2e_ms"] * 1e-3), "unit": "matvec/s",
                    "h2d_bytes_per_step": 8 * res["n_x"], "d2h_bytes_per_step": 8 * res["n_x"]},
            "gpu_launches": res["launches"],
            "clocks": res["clocks"],
            "max_rank_per_apply": res["ranks"],
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
