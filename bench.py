#!/usr/bin/env python
"""Benchmark of the GMG-preconditioned CG hot path (BASELINE.json metric
"GDoF/s of operator vmult and smoother step; GMG-CG time-to-solution +
iterations") on BASELINE.json configs[1]: 2D Poisson SIPG, k = 7, 1024^2
cells (67,108,864 dofs), 10 levels, multiplicative vertex-patch smoother with
the full kernel, fp32 V-cycle inside fp64 CG (mixed).

One "step" = one complete GMG-CG solve A x = b to ||r|| <= 1e-8 ||b|| with
f == 1 -- every row of SURVEY.md 8(a): operator apply, smoother
colour passes, residual+restriction, prolongation, coarse solve, V-cycle, PCG.
value = dofs solved per second over the timed steps (GDoF/s).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Rank 0 prints one JSON line.  --impl reference times the CPU oracle
(oracle/, numpy/scipy, 1 BLAS thread) on a bounded sample of the same workload
(the paper has no runnable reference implementation).
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = dict(name="C2", dim=2, degree=7, n_levels=10, coarse=(2, 2),
                desc="2D Poisson SIPG k=7, 1024x1024 cells, 67,108,864 dofs, 10 levels, f=1, "
                     "multiplicative full-kernel vertex-patch smoother, fp32 V-cycle / fp64 CG (BASELINE.json configs[1])")
# bounded oracle sample: same method and degree on a smaller mesh (64x64 cells)
CPU_SAMPLE = dict(dim=2, degree=7, n_levels=6)
METRIC = "GDoF/s of operator vmult and smoother step; GMG-CG time-to-solution + iterations"
UNIT = "GDoF/s (GMG-CG solve: dofs / time-to-solution)"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ---------------------------------------------------------------- roofline model
def smoother_flops_per_dof(dim, k):
    """Algorithmic flops of one full-kernel colour pass per dof (DESIGN.md
    "Roofline"), for the algorithm the kernel runs: fast diagonalisation with
    the even/odd factorised interior eigenbasis -- 2d line transforms of
    np^(d-1) lines each costing np^2/2 FMAs (two (np/2)^2 halves) + np adds,
    and one eigenvalue scaling per patch dof -- plus the face coupling (trace
    value/derivative, tangential mass, S^T M transforms, injection), counted per
    patch and divided by the patch dofs.  (The dense-eigenbasis model of
    SURVEY.md 8(d), 2d np^2 FMAs per line, is twice the FD term.)"""
    nc, np_ = k + 1, 2 * (k + 1)
    patch = np_ ** dim
    nfp = np_ ** (dim - 1)
    fd = 2 * dim * np_ ** (dim - 1) * (np_ * np_ + np_) + patch
    per_dir = 2 * nfp * 2 * nc + (dim - 1) * 2 * 2 * nfp * 2 * nc + nfp * np_ * 3
    return (fd + dim * per_dir) / patch


def alu_peak_tflops(prec, peaks):
    """CUDA-core peak from the unit counts and the max SM clock
    (B200: 148 SMs x 128 FP32 lanes, FP64 at half rate; 2 flops per FMA)."""
    mhz = peaks.get("sm_max_mhz", 1965.0)
    lanes = 128 if prec == "fp32" else 64
    return 148 * lanes * 2 * mhz * 1e6 / 1e12


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.device)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [t.strip() for t in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- distributed
def dist_init(backend):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws <= 1:
        return 0, 1, 0
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    if backend == "nccl":
        import torch
        torch.cuda.set_device(local)
    dist.init_process_group(backend)
    return rank, ws, local


# ---------------------------------------------------------------- CPU oracle leg
def oracle_sample_solve():
    """Set up the oracle on the bounded sample; returns (solve_fn, ndofs).
    Setup (assembly, patch LU factorisations) is excluded from timing, as on
    the GPU."""
    from oracle import assemble, krylov, multigrid
    V = multigrid.VCycle(CPU_SAMPLE["dim"], CPU_SAMPLE["degree"], CPU_SAMPLE["n_levels"], dtype=np.float32)
    L = CPU_SAMPLE["n_levels"] - 1
    A = V.A64[L]
    b = assemble.rhs(V.levels[L], CPU_SAMPLE["degree"])

    def solve():
        x, hist, conv = krylov.pcg(A, b, V, rtol=1e-8)
        return len(hist) - 1
    return solve, A.shape[0]


def cpu_threads_limit():
    """Pin every BLAS/OpenMP pool to 1 thread.  The libraries must be loaded
    first: threadpoolctl only limits pools that exist when it is called."""
    try:
        import scipy.linalg  # noqa: F401
        import scipy.sparse.linalg  # noqa: F401
        from oracle import multigrid  # noqa: F401
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=1)
    except Exception:
        return None


def sample_desc():
    n = 2 ** (CPU_SAMPLE["n_levels"])
    return ("oracle GMG-CG solve (numpy/scipy, fp32 V-cycle, 1 BLAS thread) on 2D k=%d, %dx%d cells, "
            "%d levels, %d dofs; setup excluded" % (CPU_SAMPLE["degree"], n, n, CPU_SAMPLE["n_levels"],
                                                    n * n * (CPU_SAMPLE["degree"] + 1) ** 2))


def run_cpu_baseline(reps=1):
    lim = cpu_threads_limit()
    solve, n = oracle_sample_solve()
    t = []
    its = 0
    for _ in range(reps):
        t0 = time.perf_counter()
        its = solve()
        t.append(time.perf_counter() - t0)
    del lim
    sec = float(np.median(t))
    return {"value": n / sec / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample_desc(),
            "seconds_per_solve": sec, "iterations": its}


def run_reference(args, rank, ws):
    if rank != 0:
        return
    lim = cpu_threads_limit()
    solve, n = oracle_sample_solve()
    for _ in range(args.warmup):
        solve()
    t0 = time.perf_counter()
    its = 0
    for _ in range(args.steps):
        its = solve()
    sec = (time.perf_counter() - t0) / args.steps
    del lim
    value = n / sec / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64 (fp32 V-cycle)", "data": "synthetic (f=1)",
            "config": {"workload": WORKLOAD["name"] + ": " + WORKLOAD["desc"], "sample": sample_desc()},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample_desc()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "iterations": its}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our CUDA path
def run_ours(args, rank, ws, local):
    import torch
    from paper_2405_18982_b200 import ipmg

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist = None
    if ws > 1:
        import torch.distributed as dist
    wl = WORKLOAD
    comm = ipmg.Comm.from_torch_distributed(local) if ws > 1 else None
    # multi-GPU: levels where a rank would keep < 1M dofs are replicated (their halo
    # exchanges would cost more NCCL latency than computing them redundantly)
    h = ipmg.Handle(wl["dim"], wl["degree"], wl["n_levels"], coarse_cells=wl["coarse"],
                    vcycle_precision=ipmg.FP32, device=local, comm=comm, dist_min_dofs=1 << 20)
    L = wl["n_levels"] - 1
    n = h.ndofs(L)                      # this rank's dofs (slab of the finest level)
    n_glob = n
    if dist:
        t = torch.tensor([n], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        n_glob = int(t.item())
    b = torch.empty(n, dtype=torch.float64, device=dev)
    h.rhs(L, b)
    x = torch.empty_like(b)
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        res = h.cg_solve(b, x, rtol=1e-8, max_it=100)
    torch.cuda.synchronize()

    # ---- timed region: K complete solves, inputs resident (537 MB > L2: no flush needed)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)
    launches0 = h.launch_count()
    h.profile(True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    its = []
    for _ in range(args.steps):
        res = h.cg_solve(b, x, rtol=1e-8, max_it=100)
        its.append(res["iterations"])
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    launches = h.launch_count() - launches0
    prof = {c: h.profile_read(c) for c in ("smooth", "vmult", "restrict", "prolong", "coarse", "blas")}
    h.profile(False)
    clk = clocks.stop()
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = n_glob / (ms_step * 1e-3) / 1e9     # strong scaling: the whole problem per step

    # ---- components (separately timed, CUDA events): vmult fp64 and one smoother step fp32
    comp = {}
    xs = torch.empty(n, dtype=torch.float64, device=dev).uniform_(-1, 1)
    ys = torch.empty_like(xs)
    for _ in range(3):
        h.vmult(L, xs, ys)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    c0.record(stream)
    for _ in range(reps):
        h.vmult(L, xs, ys)
    c1.record(stream)
    torch.cuda.synchronize()
    comp["vmult_fp64_gdofs"] = n / (c0.elapsed_time(c1) / reps * 1e-3) / 1e9
    xf, bf = xs.float(), b.float()
    for _ in range(2):
        h.smooth(L, xf, bf)
    c0.record(stream)
    for _ in range(reps):
        h.smooth(L, xf, bf)
    c1.record(stream)
    torch.cuda.synchronize()
    comp["smoother_step_fp32_gdofs"] = n / (c0.elapsed_time(c1) / reps * 1e-3) / 1e9
    del xs, ys, xf, bf

    # ---- end-to-end through the public API with host buffers (pinned): every step
    # copies its b host->device and its solution device->host.  The copies run on
    # their own streams, double-buffered, so step i's download and step i+1's
    # upload overlap the neighbouring solves (PCIe is full duplex); the events
    # order upload -> solve -> download per step and the buffer reuse.
    b_host = b.cpu().pin_memory()
    x_host = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
    bd = [torch.empty_like(b) for _ in range(2)]
    xd = [torch.empty_like(b) for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_solved = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    e2e_steps = max(2, min(args.steps, 10))
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    s_in.wait_event(e0)
    with torch.cuda.stream(s_in):
        bd[0].copy_(b_host, non_blocking=True)
        ev_in[0].record(s_in)
    for i in range(e2e_steps):
        cur, nxt = i % 2, (i + 1) % 2
        if i + 1 < e2e_steps:                      # upload of the next step's b
            if i >= 1:
                s_in.wait_event(ev_solved[nxt])    # bd[nxt] was read by solve i-1
            with torch.cuda.stream(s_in):
                bd[nxt].copy_(b_host, non_blocking=True)
                ev_in[nxt].record(s_in)
        stream.wait_event(ev_in[cur])
        if i >= 2:
            stream.wait_event(ev_out[cur])         # xd[cur] downloaded by step i-2
        h.cg_solve(bd[cur], xd[cur], rtol=1e-8, max_it=100)
        ev_solved[cur].record(stream)
        s_out.wait_event(ev_solved[cur])
        with torch.cuda.stream(s_out):
            x_host[cur].copy_(xd[cur], non_blocking=True)
            ev_out[cur].record(s_out)
    stream.wait_event(ev_out[(e2e_steps - 1) % 2])
    stream.wait_event(ev_out[e2e_steps % 2])
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    e2e_err = float((x_host[(e2e_steps - 1) % 2] - x.cpu()).abs().max() / x.abs().max().cpu())
    if dist:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    if rank != 0:
        return
    peaks, src = measured_peaks()
    # roofline of the dominant kernel: the finest-level smoother colour pass (fp32)
    nl_s, ms_s, by_s = prof["smooth"]
    avg_ms = ms_s / max(nl_s, 1)
    achieved_gbs = by_s / (ms_s * 1e-3) / 1e9 if ms_s > 0 else 0.0
    fl = smoother_flops_per_dof(wl["dim"], wl["degree"]) * n * nl_s
    achieved_tf = fl / (ms_s * 1e-3) / 1e12 if ms_s > 0 else 0.0
    hbm_peak = peaks["hbm_gbs"]
    alu_peak = alu_peak_tflops("fp32", peaks)
    t_bytes = by_s / (hbm_peak * 1e9)
    t_flops = fl / (alu_peak * 1e12)
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "smooth_traffic.json")
    if os.path.exists(tr_path):
        try:
            traffic = json.load(open(tr_path)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    if t_bytes >= t_flops:
        roof = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved_gbs / hbm_peak, "traffic": traffic}
    else:
        roof = {"bound": "alu", "achieved": achieved_tf, "peak": alu_peak, "unit": "TFLOP/s",
                "frac": achieved_tf / alu_peak, "traffic": traffic}
    roof.update({"kernel": "smooth_kernel<2,float> (k=7), finest level", "peak_source": src,
                 "launches": nl_s, "avg_launch_ms": avg_ms,
                 "algorithmic_bytes_per_launch": by_s / max(nl_s, 1),
                 "hbm_frac": achieved_gbs / hbm_peak, "alu_frac": achieved_tf / alu_peak,
                 "share_of_step": ms_s / ms if ms > 0 else None,
                 "per_class_ms_share": {c: (v[1] / ms if ms > 0 else None) for c, v in prof.items()}})
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64 CG / f32 V-cycle", "data": "synthetic (f=1 right-hand side)",
            "config": {"workload": wl["name"] + ": " + wl["desc"], "dofs": n_glob, "dofs_rank0": n,
                       "parallelism": "1 GPU" if ws == 1 else
                       "slab decomposition along y over %d ranks (NCCL halo exchange + allgathered CG scalars)" % ws,
                       "l2": "inputs larger than L2 (537 MB fp64 vectors), no flush"},
            "time_to_solution_ms": ms_step, "cg_iterations": its[-1], "nu": res["nu"],
            "components": comp, "roofline": roof, "clocks": clk, "gpu_launches": launches,
            "e2e": {"value": n_glob / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": 8 * n_glob,
                    "d2h_bytes_per_step": 8 * n_glob, "ms_per_step": e2e_ms, "steps": e2e_steps,
                    "copies": "pinned host buffers, H2D/D2H on their own streams, double-buffered "
                              "(overlapping the neighbouring steps' solves)",
                    "solution_max_rel_diff_vs_device_run": e2e_err}}
    if not args.no_cpu_baseline and ws == 1:
        line["cpu_baseline"] = run_cpu_baseline()
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        rank, ws, _ = dist_init("gloo")
        run_reference(args, rank, ws)
        return
    rank, ws, local = dist_init("nccl")
    run_ours(args, rank, ws, local)


if __name__ == "__main__":
    main()
