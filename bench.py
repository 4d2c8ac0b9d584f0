#!/usr/bin/env python
"""Benchmark of the discrete X-ray transform hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU, NCCL)

One STEP = one pass of the whole hot path over the
configuration's full ray set: the forward projection sino = A x (every ray of every view)
followed by the adjoint x' = A^T sino, i.e. one application of the normal operator
A^T A.  With N GPUs the views are split into N contiguous blocks (one plan per rank); each
rank projects its block and backprojects it into a partial image, and the partial images
are summed with one NCCL all_reduce (the path's only exchange step; x stays replicated, so
no broadcast is needed between steps).  Strong scaling: the configuration is fixed.

``value`` = rays per second of the whole job (all M rays through A and A^T per step).
``e2e``   = the same through the host-buffer C-ABI entry points (xrt_forward_host /
            xrt_adjoint_host): H2D of x and of the adjoint input, D2H of sino and x'
            inside the timed region.
``roofline`` for the dominant kernel: FP32-issue bound: algorithmic
            FP32 ops = c * nnz per launch (c = 4 in 2D, 5 in 3D; nnz counted exactly) over
            148 SMs x 128 lanes x sm_max_mhz.
``cpu_baseline``: the fp64 oracle (oracle/, as it stands) on a bounded ray sample of the same
            workload on this host's cores (rank 0, N = 1 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "forward-projection rays/s and intersections/s (plus adjoint) vs roofline, 1–8 B200"
C_OPS = {2: 4, 3: 5}  # algorithmic FP32 ops per ray-unit intersection


def peaks():
    """Roofline denominators.  HBM and the SM clock from the driver-written MEASURED_PEAKS.json; the
    FP32 issue rate from tools/issue_peak (profiles/issue_peak.json): the highest FP32 lane rate per
    SM-cycle it measured on this GPU type (packed FFMA2 / FADD2 / FMUL2 or scalar FFMA, 8 independent
    chains, 64 warps per SM) x 148 SMs x sm_max_mhz.  Fallback: the nominal 128 lanes."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    src = "measured"
    try:
        with open(path) as f:
            pk = json.load(f)
    except Exception:
        pk = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}
        src = "fallback"
    sm_mhz = float(pk.get("sm_max_mhz", 1965.0))
    lanes, lanes_src = 128.0, "nominal 128 FP32 lanes per SM-cycle (profiles/issue_peak.json missing)"
    try:
        with open(os.path.join(ROOT, "profiles", "issue_peak.json")) as f:
            ip = json.load(f)
        best = max(("FFMA", "FFMA2", "FADD2", "FMUL2"), key=lambda k: ip[k]["lane_ops_per_sm_cycle"])
        lanes = float(ip[best]["lane_ops_per_sm_cycle"])
        lanes_src = (f"measured: tools/issue_peak (profiles/issue_peak.json), {best} {lanes:.1f} FP32 lane ops "
                     f"per SM-cycle (of 128 nominal)")
    except Exception:
        pass
    return {"hbm_gbs": float(pk["hbm_gbs"]), "sm_mhz": sm_mhz, "fp32_lanes": lanes,
            "fp32_tops": 148 * lanes * sm_mhz * 1e6 / 1e12, "src": src,
            "fp32_src": f"{lanes_src} x 148 SMs x {sm_mhz:.0f} MHz ({src} sm_max_mhz, MEASURED_PEAKS.json)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}




def measured_traffic(workload: str, kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu --set full capture
    (profiles/traffic.json, written by tools/ncu_summary.py traffic); None if not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        return t[workload][kernel]["dram_bytes"]
    except Exception:
        return None


def reduction_roofline(workload: str, nnz: int, adj_ms: float):
    """The adjoint's second roofline: the SM -> L2 reduction path.  peak = the highest reduction
    sector rate tools/red_peak measured on this GPU type (profiles/red_peak.json); algorithmic
    sectors = nnz / 8 (every 32-byte sector carrying 8 units); measured sectors per launch from the
    ncu capture (profiles/traffic.json).  None when either file is missing."""
    try:
        with open(os.path.join(ROOT, "profiles", "red_peak.json")) as f:
            rp = json.load(f)
        peak = max(rp["coalesced"]["sectors_per_s"], rp["scattered"]["sectors_per_s"])
    except Exception:
        return None
    alg = nnz / 8.0
    out = {"bound": "l2_reduction", "unit": "sectors/s", "peak": peak,
           "peak_source": "tools/red_peak (profiles/red_peak.json): red.global.add.f32 from all SMs into an "
                          "L2-resident buffer, max over the coalesced and scattered patterns",
           "achieved": alg / (adj_ms / 1e3), "frac": alg / (adj_ms / 1e3) / peak,
           "algorithmic_sectors": alg}
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            rs = json.load(f)[workload]["adjoint"]["red_sectors"]
        out["measured_sectors"] = rs
        out["measured_frac"] = rs / (adj_ms / 1e3) / peak
    except Exception:
        pass
    return out


def cpu_baseline(c: dict, budget_s: float = 12.0):
    """The oracle, as it stands (fp64 brute force, mode 2: the i loop restricted to the x-range that
    can meet the (k, j) overlap -- identical output to the full loop, tested), forward, on this
    host's cores: the FULL sinogram of cfg 1 / 2, 4096 stratified rays of
    cfg 3 / 5, and a bounded (~budget_s) stratified sample of cfg 4."""
    import oracle
    from oracle import geometry as G
    img = workloads.make_image(c, device="cuda" if torch.cuda.is_available() else "cpu").cpu().numpy().reshape(-1)
    M = workloads.configs.n_rays(c)
    idx = int(c["name"][3])
    t_used, done, nnz = 0.0, 0, 0
    if idx in (1, 2, 3, 5):
        if idx in (1, 2):
            chunks = [np.arange(a, min(M, a + 200000), dtype=np.int64) for a in range(0, M, 200000)]
            what = f"the full sinogram ({M} rays)"
        else:
            chunks = [workloads.sample_rays(c, 4096, seed=9000)]
            what = f"{chunks[0].size} seeded stratified rays"
        for ids in chunks:
            p, th = G.rays(c, ids)
            t0 = time.perf_counter()
            rp, _, _ = oracle.rows(c, p, th, mode=2)
            oracle.forward(c, img, p, th, mode=2)
            t_used += time.perf_counter() - t0
            done += ids.size
            nnz += int(rp[-1])
        t_used /= 2.0   # rows + forward walk the same boxes; report one pass
    else:
        seed, batch = 9000, 64
        while t_used < budget_s and done < 200000:
            ids = workloads.sample_rays(c, batch, seed=seed)
            seed += 1
            p, th = G.rays(c, ids)
            t0 = time.perf_counter()
            oracle.forward(c, img, p, th, mode=2)
            t_used += time.perf_counter() - t0
            done += ids.size
            if t_used < budget_s / 8:
                batch *= 2
        what = f"{done} seeded stratified rays"
    out = {"value": done / t_used, "unit": "rays/s", "cores": oracle.threads(), "kind": "oracle",
           "sample": f"{what} of {c['name']}, fp64 brute-force forward (mode 2), {t_used:.1f} s",
           "full_sinogram_s_extrapolated": M / (done / t_used)}
    if nnz:
        out["intersections_per_s"] = nnz / t_used
    # context: the paper's own O(N)-per-ray enumeration on the same host cores (cpu_method/, N3)
    try:
        import cpu_method
        n = 2000000
        ids = workloads.sample_rays(c, n, seed=9500)
        p, th = G.rays(c, ids)
        cpu_method.forward(c, img, p[:1000], th[:1000])
        t0 = time.perf_counter()
        cpu_method.forward(c, img, p, th)
        dt = time.perf_counter() - t0
        out["paper_method_cpu"] = {"value": n / dt, "unit": "rays/s", "cores": cpu_method.threads(),
                                   "sample": f"{n} seeded rays of {c['name']}, fp64 incremental enumeration "
                                             f"(Algorithm 3.1), {dt:.2f} s"}
    except Exception as e:  # context only
        out["paper_method_cpu"] = {"value": None, "error": str(e)}
    return out


def run_reference(args, c, rank, world):
    """--impl reference: the oracle as the reference arm (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    from oracle import geometry as G
    img = workloads.make_image(c, device="cuda" if torch.cuda.is_available() else "cpu").cpu().numpy().reshape(-1)
    per_step = args.ref_rays
    times = []
    seed = 7000
    for s in range(args.warmup + args.steps):
        ids = workloads.sample_rays(c, per_step, seed=seed + s)
        p, th = G.rays(c, ids)
        y = np.ones(ids.size)
        t0 = time.perf_counter()
        oracle.forward(c, img, p, th)
        oracle.adjoint(c, y, p, th)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append((ids.size, dt))
    rays = sum(n for n, _ in times)
    tt = sum(t for _, t in times)
    val = rays / tt
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "rays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tt / max(1, len(times)),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": c["name"], "rays_per_step": per_step,
                                            "note": "each reference step = forward + adjoint of a seeded ray sample"},
            "cpu_baseline": {"value": val, "unit": "rays/s", "cores": oracle.threads(), "kind": "oracle",
                             "sample": f"{per_step} seeded rays per step, fp64 brute force (forward + adjoint)"},
            "e2e": {"value": val, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--algo", default="auto", choices=["auto", "ray", "column"])
    ap.add_argument("--adj-algo", default=None, choices=["auto", "ray", "column", "gather"],
                    help="adjoint kernel family (default: --algo)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-attenuated", action="store_true",
                    help="skip the attenuated-transform side measurement (SURVEY 8(f) N4)")
    ap.add_argument("--ref-rays", type=int, default=256)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: functional check of the N > 1 step with fewer GPUs than ranks (ranks share "
                         "GPUs, collectives through the host; no kernel waits on another rank) -- not a "
                         "measurement")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    c = workloads.config(args.config)
    if args.impl == "reference":
        run_reference(args, c, rank, world)
        return

    if args.dist_backend == "gloo":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    from paper_2006_00686_b200 import Plan
    from paper_2006_00686_b200.dist import ShardedPlan

    sp = ShardedPlan(c, rank=rank, world=world, device=local)
    plan: Plan = sp.plan
    if args.algo != "auto":
        plan.set_algorithm("forward", args.algo)
        plan.set_algorithm("adjoint", args.algo)
    if args.adj_algo is not None:
        plan.set_algorithm("adjoint", args.adj_algo)
    x = workloads.make_image(c, device=dev)
    sino = torch.empty(plan.sino_shape, dtype=torch.float32, device=dev)
    xo = torch.empty_like(x)
    nnz_local = plan.n_units
    nnz = torch.tensor([nnz_local], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(nnz)
    nnz_total = int(nnz.item())
    M = workloads.configs.n_rays(c)
    dim = 2 if c["beam"] in ("par2d", "fan2d") else 3
    s = torch.cuda.current_stream()
    helical_windows = world > 1 and c["beam"] == "helical"

    def step(ev=None):
        """One pass of the hot path: (N > 1: x to every rank -- broadcast, or the helical z windows)
        A x over this rank's views, then A^T over them (+ the overlapped staged all-reduce, or the
        helical window exchange)."""
        if ev is not None:
            ev[0].record(s)
        if world > 1:
            if helical_windows:
                sp.scatter_windows(x, src=0)
            else:
                dist.broadcast(x, src=0)
        if ev is not None:
            ev[1].record(s)
        plan.forward(x, out=sino)
        if ev is not None:
            ev[2].record(s)
        if helical_windows:
            sp.adjoint_windowed(sino, out=xo)
        else:
            sp.adjoint(sino, out=xo, overlap=True)
        if ev is not None:
            ev[3].record(s)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    launches0 = plan.launch_count
    with ClockSampler(local) as clk:
        start.record(s)
        for k in range(args.steps):
            step(evs[k])
        end.record(s)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = plan.launch_count - launches0
    ms = start.elapsed_time(end)
    step_ms = [e[0].elapsed_time(e[3]) for e in evs]
    bc_ms = [e[0].elapsed_time(e[1]) for e in evs]
    fwd_ms = [e[1].elapsed_time(e[2]) for e in evs]
    adj_ms = [e[2].elapsed_time(e[3]) for e in evs]     # adjoint (+ its overlapped reduction for N > 1)
    t = torch.tensor([ms, sum(fwd_ms), sum(adj_ms), sum(bc_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, fwd_sum, adj_sum, bc_sum = [float(v) for v in t.tolist()]
    value = M * args.steps / (ms_max / 1e3)
    # the adjoint kernels alone (no collective), for the compute / collective split at N > 1
    adj_compute_ms = None
    if world > 1:
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a0.record(s)
        for _ in range(args.steps):
            plan.adjoint(sino, out=xo)
        a1.record(s)
        torch.cuda.synchronize()
        ta = torch.tensor([a0.elapsed_time(a1) / args.steps], dtype=torch.float64, device=dev)
        dist.all_reduce(ta, op=dist.ReduceOp.MAX)
        adj_compute_ms = float(ta.item())

    # ---------------- e2e: host buffers in, host buffers out, through the public API
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        sh = torch.empty(plan.sino_shape, dtype=torch.float32).pin_memory()
        xoh = torch.empty(plan.image_shape, dtype=torch.float32).pin_memory()

        def e2e_step():
            if world == 1:
                # the C ABI's host-buffer entry points (copies pipelined with the kernels inside)
                plan.forward_host(xh, out=sh)
                plan.adjoint_host(sh, out=xoh)
            else:
                # sharded: H2D of x, A x, D2H of this rank's sinogram slab; H2D of the slab, A^T with
                # the overlapped all-reduce, D2H of the image
                x.copy_(xh, non_blocking=True)
                plan.forward(x, out=sino)
                sh.copy_(sino, non_blocking=True)
                sino.copy_(sh, non_blocking=True)
                if helical_windows:
                    sp.adjoint_windowed(sino, out=xo)
                else:
                    sp.adjoint(sino, out=xo, overlap=True)
                xoh.copy_(xo, non_blocking=True)
        e2e_step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ke = max(1, min(args.steps, 3))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(ke):
            e2e_step()
        e1.record(s)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te.item())
        img_b = x.numel() * 4
        sino_b = sino.numel() * 4
        e2e = {"value": M * ke / (e2e_ms / 1e3), "unit": "rays/s", "ms_per_step": e2e_ms / ke,
               "h2d_bytes_per_step": img_b + sino_b, "d2h_bytes_per_step": sino_b + img_b,
               "note": ("xrt_forward_host + xrt_adjoint_host (copies pipelined inside the C ABI)" if world == 1 else
                        "ShardedPlan: H2D x, A x, D2H + H2D of the rank's sinogram slab, A^T with the "
                        "overlapped all-reduce, D2H image") + "; pinned host buffers; bytes per rank"}

    # ---------------- attenuated transform (N4): side measurement, outside the timed step
    att = None
    if world == 1 and not args.no_attenuated:
        mu = workloads.make_attenuation(c, device=dev)
        y = sino.clone()

        def att_ms(fn, reps=2):
            fn()
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(s)
            for _ in range(reps):
                fn()
            a1.record(s)
            torch.cuda.synchronize()
            return a0.elapsed_time(a1) / reps

        la0 = plan.launch_count
        f_ms = att_ms(lambda: plan.forward_attenuated(x, mu, out=sino))
        b_ms = att_ms(lambda: plan.adjoint_attenuated(y, mu, out=xo))
        att = {"forward_ms": f_ms, "adjoint_ms": b_ms,
               "forward_rays_per_s": M / (f_ms / 1e3), "adjoint_rays_per_s": M / (b_ms / 1e3),
               "forward_intersections_per_s": nnz_local / (f_ms / 1e3),
               "gpu_launches": plan.launch_count - la0,
               "note": "xrt_forward_attenuated / xrt_adjoint_attenuated (SPECT weight, DESIGN reading 23), "
                       "column kernels on the 3D beams (untiled) else RAY, mu = workloads.make_attenuation; "
                       "1 warm-up + 2 timed calls each, not in the step"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    pk = peaks()
    c_ops = C_OPS[dim]
    fwd_avg = fwd_sum / args.steps
    adj_avg = adj_sum / args.steps if world == 1 else adj_compute_ms
    # per-rank kernels: ops of this rank's shard
    k_fwd = {"ms": fwd_avg, "tflops": c_ops * nnz_local / (fwd_avg / 1e3) / 1e12}
    k_adj = {"ms": adj_avg, "tflops": c_ops * nnz_local / (adj_avg / 1e3) / 1e12}
    dom_name, dom = ("adjoint", k_adj) if adj_avg >= fwd_avg else ("forward", k_fwd)
    roof = {"bound": "alu", "kernel": dom_name, "achieved": dom["tflops"], "peak": pk["fp32_tops"],
            "unit": "TFLOP/s", "frac": dom["tflops"] / pk["fp32_tops"],
            "traffic": measured_traffic(c["name"], dom_name) if world == 1 else None,
            "traffic_unit": "bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, ncu --set full)",
            "algorithmic_bytes": int(4 * (x.numel() + sino.numel())),
            "peak_source": pk["fp32_src"],
            "ops_per_intersection": c_ops}
    line = {
        "metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "ms_per_step_median": statistics.median(step_ms), "ms_per_step_min": min(step_ms),
        "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": c["name"], "rays": M, "intersections": nnz_total,
                   "image": list(c["n"]), "views": c["n_views"], "det": [c["det_rows"], c["det_cols"]],
                   "step": "sino = A x; x' = A^T sino (N > 1: broadcast x, staged all-reduce of x' overlapped "
                           "with the adjoint; helical: z-window scatter / P2P overlap exchange)",
                   "l2": "inputs larger than L2 (image + sinogram > 126 MB)" if (x.numel() + sino.numel()) * 4 > 126e6
                   else "inputs smaller than L2 (no flush)",
                   "parallelism": f"views/{world}",
                   **({"dist_backend": args.dist_backend + (" (functional check, ranks share GPUs: not a "
                                                            "measurement)" if args.dist_backend == "gloo" else "")}
                      if world > 1 else {})},
        "intersections_per_s": nnz_total * args.steps / (ms_max / 1e3),
        "forward": {"ms": fwd_avg, "ms_median": statistics.median(fwd_ms), "ms_min": min(fwd_ms),
                    "rays_per_s": M / world / (fwd_avg / 1e3),
                    "intersections_per_s": nnz_local / (fwd_avg / 1e3),
                    "roofline_frac": k_fwd["tflops"] / pk["fp32_tops"]},
        "adjoint": {"ms": adj_avg, "ms_median": statistics.median(adj_ms) if world == 1 else adj_compute_ms,
                    "ms_min": min(adj_ms) if world == 1 else adj_compute_ms,
                    "rays_per_s": M / world / (adj_avg / 1e3),
                    "intersections_per_s": nnz_local / (adj_avg / 1e3),
                    "roofline_frac": k_adj["tflops"] / pk["fp32_tops"]},
        "roofline": roof,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "algo": args.algo, "adj_algo": args.adj_algo or args.algo,
    }
    if world > 1:
        line["collective"] = {
            "broadcast_ms": bc_sum / args.steps, "forward_ms": fwd_avg,
            "adjoint_plus_reduce_ms": adj_sum / args.steps, "adjoint_compute_ms": adj_compute_ms,
            "exposed_reduce_ms": adj_sum / args.steps - adj_compute_ms,
            "mode": "helical z windows (scatter + P2P overlaps)" if helical_windows else
                    "broadcast + staged all-reduce overlapped with the adjoint bands",
            "note": "max over ranks; compute-only = the adjoint kernels timed alone"}
    if world == 1 and args.adj_algo in (None, "auto", "column") and args.algo in ("auto", "column") and dim == 3:
        rr = reduction_roofline(c["name"], nnz_local, adj_avg)
        if rr is not None:
            line["adjoint"]["roofline_reduction"] = rr
    if e2e is not None:
        line["e2e"] = e2e
    if att is not None:
        line["attenuated"] = att
    if world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline(c)
        except Exception as e:  # never let the baseline kill the bench line
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
