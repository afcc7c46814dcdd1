#!/usr/bin/env python
"""Benchmark of the B200 FP64 TT hot path (BASELINE.json metric, config 5 = W5 workload).

One step = the whole hot path over one batch of synthetic config-5 input, through the C-ABI:
  tt_sweep_als   (H1-H7: initial right interfaces, L->R sweep with K=32 batched local
                  matvecs + left interfaces, R->L sweep with batched matvecs + right
                  interfaces; DESIGN.md §5 workload W5)
  tt_operator_apply (H8: full unrounded TT-matrix x TT-vector product)
Value = algorithmic FP64 GFLOP per step / device time per step (CUDA events, max over ranks).

  python bench.py [--gpus N --steps K --warmup W]          # our CUDA path
  python bench.py --impl reference [--steps K --warmup W]  # the CPU oracle, as it stands

Multi-GPU: replicas only — each rank runs the same workload, no collective on
the data path; the barrier/all-reduce below is timing plumbing.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import ttgen  # noqa: E402

METRIC = "FP64 GFLOP/s + % FP64 roofline of TT local matvec; full-sweep time at d=12"
UNIT = "GFLOP/s"


# ----------------------------------------------------------------------------------------
# algorithmic work
# ----------------------------------------------------------------------------------------
def f_local(a, N, b, al, be):
    """FLOPs of one local matvec (per vector) == one interface update: three products."""
    return 2 * N * (a * a * al * b + a * b * b * be) + 2 * a * b * al * be * N * N


def b_local_matvec(a, N, b, al, be, K):
    return 8 * (a * a * al + b * b * be + al * N * N * be + 2 * K * a * N * b)


def f_apply(a, N, b, al, be):
    return 2 * a * al * N * b * be * N


def b_apply(a, N, b, al, be):
    return 8 * (a * N * b + al * N * N * be + a * al * N * b * be)


def w5_work(cfg):
    d, N, r, R, K = cfg.d, cfg.N, cfg.r, cfg.R, cfg.nvec
    mv = sum(2 * K * f_local(r[k], N, r[k + 1], R[k], R[k + 1]) for k in range(d))
    iface = sum(f_local(r[k], N, r[k + 1], R[k], R[k + 1]) for k in range(1, d)) * 2 \
        + sum(f_local(r[k], N, r[k + 1], R[k], R[k + 1]) for k in range(0, d - 1))
    ap = sum(f_apply(r[k], N, r[k + 1], R[k], R[k + 1]) for k in range(d))
    ap_bytes = sum(b_apply(r[k], N, r[k + 1], R[k], R[k + 1]) for k in range(d))
    return {"matvec_flops": mv, "interface_flops": iface, "apply_flops": ap,
            "apply_bytes": ap_bytes, "step_flops": mv + iface + ap}


# ----------------------------------------------------------------------------------------
# multi-rank plumbing (replicas only: no collective on the data path)
# ----------------------------------------------------------------------------------------
def max_over_ranks(ms: float, device) -> float:
    """Max of a per-rank device time over all ranks (timing plumbing; identity at N=1)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return ms
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(work_per_step: float, world: int, steps: int, max_ms: float) -> float:
    """Whole-job throughput: all ranks' work / the slowest rank's time (GFLOP/s)."""
    return work_per_step * world * steps / (max_ms * 1e-3) / 1e9


def bench_w34_flops(cfg):
    """W34 = (d-1) right + (d-1) left interface updates + one local matvec per core."""
    d, N, r, R = cfg.d, cfg.N, cfg.r, cfg.R
    f = [f_local(r[k], N, r[k + 1], R[k], R[k + 1]) for k in range(d)]
    return sum(f[1:]) + sum(f[:-1]) + sum(f)


def w34_executed_flops(cfg):
    """FLOPs tt_sweep_w34 executes: d left and d right interface updates (the chains include
    the boundary updates giving x^T A x) and, per core, only the matvec's last stage — its first
    two stages are the left update's (same phiL[k], A_k, x_k with K = 1), whose T2_k is kept."""
    d, N, r, R = cfg.d, cfg.N, cfg.r, cfg.R
    f = [f_local(r[k], N, r[k + 1], R[k], R[k + 1]) for k in range(d)]
    s3 = [2.0 * r[k] * N * r[k + 1] ** 2 * R[k + 1] for k in range(d)]
    return 2 * sum(f) + sum(s3)


def time_sweep(tt, fn, stream, dev, reps=5):
    """Median/best device time of `fn` run eagerly and replayed from a captured CUDA graph."""
    import torch
    fn(stream)
    torch.cuda.synchronize(dev)
    eager = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn(stream)
        e1.record(stream)
        e1.synchronize()
        eager.append(e0.elapsed_time(e1))
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(dev)
    cap.wait_stream(stream)
    with torch.cuda.stream(cap):
        with torch.cuda.graph(graph, stream=cap):
            fn(cap)
    torch.cuda.synchronize(dev)
    graphed = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        graph.replay()
        e1.record(stream)
        e1.synchronize()
        graphed.append(e0.elapsed_time(e1))
    return {"eager_ms_median": statistics.median(eager), "eager_ms_best": min(eager),
            "graph_ms_median": statistics.median(graphed), "graph_ms_best": min(graphed)}


# ----------------------------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(p[1]) for p in rows if p[1].replace(".", "").isdigit()]
        smax = [float(p[2]) for p in rows if p[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for p in rows for i in range(4) if "Active" in p[5 + i]
                          and "Not" not in p[5 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------------------------------------
# reference arm: the CPU oracle as it stands
# ----------------------------------------------------------------------------------------
def oracle_sample_inputs(seed=7):
    """Config-5 interior-core shapes (a=b=256, alpha=beta=36, N=4), seeded random values."""
    cfg = ttgen.CONFIGS[5]
    k = 6
    a, b, al, be, N = cfg.r[k], cfg.r[k + 1], cfg.R[k], cfg.R[k + 1], cfg.N
    rng = np.random.default_rng(seed)
    return dict(a=a, b=b, al=al, be=be, N=N,
                phiL=rng.standard_normal((a, al, a)), A=rng.standard_normal((al, N, N, be)),
                phiR=rng.standard_normal((b, be, b)), x=rng.standard_normal((a, N, b)))


class pinned_one_core:
    """the oracle is timed single-threaded, pinned to one core."""
    def __enter__(self):
        self.prev = None
        try:
            self.prev = os.sched_getaffinity(0)
            self.core = max(self.prev)
            os.sched_setaffinity(0, {self.core})
        except (AttributeError, OSError):
            self.core = None
        return self

    def __exit__(self, *exc):
        if self.prev is not None:
            os.sched_setaffinity(0, self.prev)
        return False


def time_oracle_sample(with_interface=True):
    import oracle
    s = oracle_sample_inputs()
    oracle.build()
    t0 = time.perf_counter()
    oracle.local_matvec(s["phiL"], s["A"], s["phiR"], s["x"])
    flops = f_local(s["a"], s["N"], s["b"], s["al"], s["be"])
    if with_interface:
        oracle.interface_left(s["phiL"], s["A"], s["x"])
        flops += f_local(s["a"], s["N"], s["b"], s["al"], s["be"])
    dt = time.perf_counter() - t0
    return flops, dt


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args, rank):
    if rank != 0:
        return
    import oracle
    oracle.build()
    s = oracle_sample_inputs()
    flops = f_local(s["a"], s["N"], s["b"], s["al"], s["be"])
    with pinned_one_core() as pin:
        for _ in range(args.warmup):
            oracle.local_matvec(s["phiL"], s["A"], s["phiR"], s["x"])
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            oracle.local_matvec(s["phiL"], s["A"], s["phiR"], s["x"])
            times.append(time.perf_counter() - t0)
    total = sum(times)
    value = flops * args.steps / total / 1e9
    sample = ("one Krylov column of the config-5 interior-core (k=6: a=b=256, alpha=beta=36, N=4) "
              "local matvec per step, tt_oracle_local_matvec, seeded random interfaces")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config 5 (d=12, r=256, R=36, K=32) W5 - bounded oracle sample",
                   "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": sample, "cpu": cpu_model(), "compiler": "gcc -O2 -std=c99",
                         "pinned_core": pin.core},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-apply", action="store_true", help="debug: skip H8 in the step")
    ap.add_argument("--no-sweeps", action="store_true", help="skip the d=12 sweep timings")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--variant", type=int, default=-1, help="GEMM tiling variant (benchmark hook)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    if world > 1:
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    import paper_2509_11890_b200 as tt
    tt.tt_debug_set_variant(args.variant)

    cfg = ttgen.CONFIGS[args.config]
    work = w5_work(cfg)
    if args.no_apply:
        work["step_flops"] -= work["apply_flops"]
    inp = ttgen.make_inputs(args.config, with_block=True)
    d = cfg.d
    stream = torch.cuda.current_stream(dev)

    # pinned host copies (e2e source) and resident device copies
    def pin(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory()

    hx = [pin(c) for c in inp.x]
    hA = [pin(c) for c in inp.A]
    hX = [pin(c) for c in inp.X]
    xs = [t.to(dev) for t in hx]
    As = [t.to(dev) for t in hA]
    Xs = [t.to(dev) for t in hX]
    Yf = [torch.empty_like(X) for X in Xs]
    phiL = tt.alloc_interfaces(xs, As)
    phiR = tt.alloc_interfaces(xs, As)
    tr = tt._Train(xs, As)
    ws = torch.empty(tt.tt_sweep_als_workspace_size(tr, cfg.nvec), dtype=torch.uint8, device=dev)
    zs = None
    if not args.no_apply:
        zs = [torch.empty((cfg.r[k] * cfg.R[k], cfg.N, cfg.r[k + 1] * cfg.R[k + 1]),
                          dtype=torch.float64, device=dev) for k in range(d)]
    hY = [torch.empty(Y.shape, dtype=torch.float64).pin_memory() for Y in Yf]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2

    launches = [0]

    def step(bx=None, bA=None, bX=None, bY=None):
        bx, bA, bX, bY = bx or xs, bA or As, bX or Xs, bY or Yf
        tt.tt_sweep_als(bx, bA, bX, bY, None, phiL, phiR, workspace=ws, stream=stream)
        n = tt.tt_last_launch_count()
        if zs is not None:
            tt.tt_operator_apply(bx, bA, zs, stream=stream)
            n += tt.tt_last_launch_count()
        launches[0] += n

    # ---- FP64 peak probe (roofline denominator, measured in this run) ------------------
    def probe(iters):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fl = tt.tt_fp64_peak_probe(iters, stream=stream)
        e1.record(stream)
        e1.synchronize()
        return fl / (e0.elapsed_time(e1) * 1e-3) / 1e12

    probe(2000)
    p64_burst = max(probe(40000) for _ in range(3))          # ~20 ms each
    p64_sustained = probe(2000000)                             # ~1 s back to back

    # ---- warm-up ----------------------------------------------------------------------
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # ---- timed region -----------------------------------------------------------------
    tt.tt_trace_enable(400 * (args.steps + 1))
    clocks = ClockSampler(local_rank)
    clocks.start()
    launches[0] = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()   # L2 flush between timed steps, outside the step's events
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    clk = clocks.stop()
    gpu_launches = launches[0]
    recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
    tt.tt_trace_disable()

    total_ms = max_over_ranks(sum(step_ms), dev)
    ms_per_step = total_ms / args.steps
    value = whole_job_rate(work["step_flops"], world, args.steps, total_ms)

    # ---- per-stage breakdown from the trace -----------------------------------------------
    stages = {}
    for r in recs:
        s = stages.setdefault(r["stage"], {"launches": 0, "ms": 0.0, "flops": 0.0})
        s["launches"] += 1
        s["ms"] += r["ms"]
        if r["stage"].startswith(("mv_", "il_", "ir_")):
            s["flops"] += 2.0 * r["M"] * r["N"] * r["K"]
        elif r["stage"] == "apply":
            s["flops"] += 2.0 * r["M"] * r["N"]
    traced_ms = sum(s["ms"] for s in stages.values())
    for s in stages.values():
        s["ms_per_step"] = s["ms"] / args.steps
        s["tflops"] = s["flops"] / (s["ms"] * 1e-3) / 1e12 if s["ms"] > 0 else None
        s["share"] = s["ms"] / traced_ms if traced_ms else None
    dom_name = max((n for n in stages if n != "apply"), key=lambda n: stages[n]["ms"])
    dom = stages[dom_name]
    mv_ms = sum(stages[n]["ms"] for n in ("mv_s1", "mv_s2", "mv_s3") if n in stages)
    mv_flops = sum(stages[n]["flops"] for n in ("mv_s1", "mv_s2", "mv_s3") if n in stages)
    mv_tf = mv_flops / (mv_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(dom_name)
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "kernel": f"dmma_gemm ({dom_name})",
                "achieved": dom["tflops"], "peak": p64_sustained, "unit": "TFLOP/s",
                "frac": dom["tflops"] / p64_sustained, "traffic": traffic,
                "peak_source": "FP64 DMMA probe kernel, measured in this run (sustained ~1 s); "
                               "MEASURED_PEAKS.json has no FP64 entry",
                "peak_burst": p64_burst,
                # second line against the datasheet (HGX B200: 296 TFLOP/s
                # FP64 Tensor Core per 8 GPUs = 37 per GPU)
                "datasheet_peak": 37.0,
                "frac_vs_datasheet": dom["tflops"] / 37.0}
    apply_detail = None
    if "apply" in stages:
        ap_ms = stages["apply"]["ms"] / args.steps
        apply_detail = {"ms_per_step": ap_ms, "bytes": work["apply_bytes"],
                        "gbs": work["apply_bytes"] / (ap_ms * 1e-3) / 1e9}

    # ---- end to end through the public API from pinned host buffers ---------------------
    # Every step copies its inputs (x, A, Krylov block) host->device and its result (the Y
    # blocks) device->host inside the timed region.  The copies are double-buffered on two
    # copy streams so that step i+1's upload and step i's download overlap step i's compute.
    e2e = None
    if not args.no_e2e:
        h2d = sum(t.numel() * 8 for t in hx + hA + hX)
        d2h = sum(t.numel() * 8 for t in hY)
        sets = [(xs, As, Xs, Yf),
                ([torch.empty_like(t) for t in xs], [torch.empty_like(t) for t in As],
                 [torch.empty_like(t) for t in Xs], [torch.empty_like(t) for t in Yf])]
        hYs = [hY, [torch.empty(Y.shape, dtype=torch.float64).pin_memory() for Y in Yf]]
        up, down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev = lambda: torch.cuda.Event()
        in_ready = [ev(), ev()]
        done = [ev(), ev()]
        out_done = [ev(), ev()]

        def upload(i):
            bx, bA, bX, _ = sets[i % 2]
            with torch.cuda.stream(up):
                if i >= 2:
                    up.wait_event(done[i % 2])        # step i-2 finished reading this set
                for src, dst in zip(hx + hA + hX, bx + bA + bX):
                    dst.copy_(src, non_blocking=True)
                in_ready[i % 2].record(up)

        def run(i, nsteps):
            bx, bA, bX, bY = sets[i % 2]
            stream.wait_event(in_ready[i % 2])
            if i >= 2:
                stream.wait_event(out_done[i % 2])   # step i-2's Y has been downloaded
            step(bx, bA, bX, bY)
            done[i % 2].record(stream)
            if i + 1 < nsteps:
                upload(i + 1)
            with torch.cuda.stream(down):
                down.wait_event(done[i % 2])
                for src, dst in zip(bY, hYs[i % 2]):
                    dst.copy_(src, non_blocking=True)
                out_done[i % 2].record(down)

        upload(0)
        for i in range(2):                             # warm-up of the pipelined path
            run(i, 2)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        up.wait_stream(stream)
        down.wait_stream(stream)
        upload(0)
        for i in range(args.steps):
            run(i, args.steps)
        stream.wait_event(out_done[(args.steps - 1) % 2])
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e_ms = max_over_ranks(e0.elapsed_time(e1), dev)
        e2e = {"value": whole_job_rate(work["step_flops"], world, args.steps, e_ms),
               "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": e_ms / args.steps,
               "note": "H2D of x, A and the Krylov block and D2H of the Y blocks every step, "
                       "double-buffered on two copy streams (overlapping compute)"}

    # ---- local GMRES on the interior core (m = 10, one cycle) ----------
    gm = None
    if not args.no_sweeps:
        k = cfg.d // 2
        m_g = 10
        rl, nn, rr = cfg.r[k], cfg.N, cfg.r[k + 1]
        Rl, Rr = cfg.R[k], cfg.R[k + 1]
        Fg = Xs[k]
        Xg = torch.zeros_like(Fg)
        wsg = torch.empty(tt.tt_local_gmres_workspace_size(rl, nn, rr, Rl, Rr, cfg.nvec, m_g),
                          dtype=torch.uint8, device=dev)
        relg = torch.empty(cfg.nvec, dtype=torch.float64, device=dev)
        itg = torch.empty(cfg.nvec, dtype=torch.int64, device=dev)

        def gmres_run(st):
            Xg.zero_()
            tt.tt_local_gmres(phiL[k], As[k], phiR[k + 1], Fg, Xg, m=m_g, cycles=1, tol=0.0,
                              rel_res=relg, iters=itg, workspace=wsg, stream=st)
        t = time_sweep(tt, gmres_run, stream, dev, reps=3)
        mv_f = (m_g + 1) * cfg.nvec * f_local(rl, nn, rr, Rl, Rr)
        S = rl * nn * cfg.nvec * rr
        orth_f = sum(2 * 2 * 2 * (i + 1) * S for i in range(m_g))   # CGS2: 2 passes x (dot + axpy)
        gm = {"core": k, "nvec": cfg.nvec, "m": m_g, "cycles": 1,
              "ms": t["graph_ms_median"], "ms_eager": t["eager_ms_median"],
              "gflop": (mv_f + orth_f) / 1e9,
              "tflops": (mv_f + orth_f) / (t["graph_ms_median"] * 1e-3) / 1e12,
              "matvec_share_of_flops": mv_f / (mv_f + orth_f),
              "frac_of_p64": (mv_f + orth_f) / (t["graph_ms_median"] * 1e-3) / 1e12 / p64_sustained}

    # ---- SURVEY 8(f) rows 2 and 4 on the interior core: KKT block action, two-site matvec --
    kkt = two = None
    if not args.no_sweeps:
        k = cfg.d // 2
        rl, nn, rr = cfg.r[k], cfg.N, cfg.r[k + 1]
        Rl, Rr = cfg.R[k], cfg.R[k + 1]
        gen = torch.Generator(device=dev).manual_seed(11)
        rnd = lambda *sh: torch.randn(*sh, dtype=torch.float64, device=dev, generator=gen)
        ops = [(rnd(rl, Rl, rl), rnd(Rl, nn, nn, Rr), rnd(rr, Rr, rr)) for _ in range(8)]
        terms = [(0, 0, 0, -1, -1.0), (0, 1, 1, -1, 1.0), (1, 0, 2, -1, -1.0),
                 (1, 2, 3, -1, 1.0), (2, 0, 4, -1, 1.0), (2, 1, 5, 6, 1.0), (2, 2, 5, 7, 1.0)]
        Xk = rnd(rl, nn, 3, rr)
        Yk = torch.empty_like(Xk)
        wsk = torch.empty(tt.tt_block_local_matvec_workspace_size(rl, nn, rr, [Rl] * 8, [Rr] * 8),
                          dtype=torch.uint8, device=dev)
        t = time_sweep(tt, lambda st: tt.tt_block_local_matvec(ops, terms, Xk, Yk, workspace=wsk,
                                                              stream=st), stream, dev, reps=5)
        f9 = 9 * f_local(rl, nn, rr, Rl, Rr)
        kkt = {"core": k, "operators": 8, "terms": len(terms), "matvecs": 9,
               "ms": t["graph_ms_median"], "gflop": f9 / 1e9,
               "tflops": f9 / (t["graph_ms_median"] * 1e-3) / 1e12,
               "frac_of_p64": f9 / (t["graph_ms_median"] * 1e-3) / 1e12 / p64_sustained}
        # two-site (DMRG supercore) matvec: 2x2 modes (N = 4), bonds of the interior core
        A1, A2 = rnd(Rl, 2, 2, Rl), rnd(Rl, 2, 2, Rr)
        W2 = rnd(rl, 2, 2, cfg.nvec, rr)
        Y2 = torch.empty_like(W2)
        ws2 = torch.empty(tt.tt_local_matvec_two_site_workspace_size(rl, 2, 2, rr, Rl, Rl, Rr,
                                                                     cfg.nvec),
                          dtype=torch.uint8, device=dev)
        t = time_sweep(tt, lambda st: tt.tt_local_matvec_two_site(phiL[k], A1, A2, phiR[k + 1], W2,
                                                                  Y2, workspace=ws2, stream=st),
                       stream, dev, reps=5)
        f2 = cfg.nvec * f_local(rl, 4, rr, Rl, Rr)
        two = {"core": k, "n1": 2, "n2": 2, "nvec": cfg.nvec, "ms": t["graph_ms_median"],
               "gflop": f2 / 1e9, "tflops": f2 / (t["graph_ms_median"] * 1e-3) / 1e12,
               "frac_of_p64": f2 / (t["graph_ms_median"] * 1e-3) / 1e12 / p64_sustained}

    # ---- block LOBPCG of the step-length eigenproblem (interior core) ---
    lob = None
    if not args.no_sweeps:
        k = cfg.d // 2
        rl, nn, rr = cfg.r[k], cfg.N, cfg.r[k + 1]
        Rl, Rr = cfg.R[k], cfg.R[k + 1]
        gen = torch.Generator(device=dev).manual_seed(12)
        rnd = lambda *sh: torch.randn(*sh, dtype=torch.float64, device=dev, generator=gen)
        sym_if = lambda r, R: (lambda t: (t + t.transpose(0, 2)) / 2)(rnd(r, R, r))
        sym_core = lambda: (lambda t: (t + t.transpose(1, 2)) / 2)(rnd(Rl, nn, nn, Rr))
        opA = (sym_if(rl, Rl), sym_core(), sym_if(rr, Rr))
        # L_B = I + 0.01 (symmetric perturbation): SPD, operator ranks as the interior core's
        pLB, ALB, pRB = 0.1 * sym_if(rl, Rl), 0.1 * sym_core(), 0.1 * sym_if(rr, Rr)
        pLB[:, 0, :] += torch.eye(rl, dtype=torch.float64, device=dev)
        pRB[:, 0, :] += torch.eye(rr, dtype=torch.float64, device=dev)
        ALB[0, :, :, 0] = torch.eye(nn, dtype=torch.float64, device=dev)
        ALB[0, :, :, 1:] = 0.0
        ALB[1:, :, :, 0] = 0.0
        opB = (pLB, ALB, pRB)
        nb_l, its_l = 8, 20
        lob = {"core": k, "nb": nb_l, "iterations": its_l, "refresh": 20}
        for name, oB in (("standard", None), ("generalised", opB)):
            X0 = rnd(rl, nn, nb_l, rr)
            Xl = X0.clone()
            RlB, RrB = (Rl, Rr) if oB is not None else (0, 0)
            wsl = torch.empty(tt.tt_local_lobpcg_workspace_size(rl, nn, rr, Rl, Rr, RlB, RrB, nb_l),
                              dtype=torch.uint8, device=dev)
            bufs = [torch.empty(nb_l, dtype=torch.float64, device=dev) for _ in range(2)]
            itl = torch.empty(1, dtype=torch.int64, device=dev)
            stl = torch.empty(1, dtype=torch.float64, device=dev)

            def lob_run(st, oB=oB, Xl=Xl, X0=X0, wsl=wsl, bufs=bufs, itl=itl, stl=stl):
                Xl.copy_(X0)
                tt.tt_local_lobpcg(opA, Xl, opB=oB, maxiter=its_l, tol=0.0, lam=bufs[0],
                                   res=bufs[1], iters=itl, step=stl, workspace=wsl, stream=st,
                                   refresh=20)
            t = time_sweep(tt, lob_run, stream, dev, reps=3)
            nops = 2 if oB is not None else 1
            # matvecs: initial (1 block), one per iteration, refresh (2 blocks) every 20
            nblocks = 1 + its_l + 2 * ((its_l - 1) // 20)
            mv_f = nops * nblocks * nb_l * f_local(rl, nn, rr, Rl, Rr)
            lob[name] = {"ms": t["graph_ms_median"], "ms_eager": t["eager_ms_median"],
                         "ms_per_iteration": t["graph_ms_median"] / its_l,
                         "matvec_gflop": mv_f / 1e9,
                         "matvec_tflops_over_total_time": mv_f / (t["graph_ms_median"] * 1e-3) / 1e12,
                         "frac_of_p64": mv_f / (t["graph_ms_median"] * 1e-3) / 1e12 / p64_sustained}

    # ---- TT rounding of the config-5 vector train (delta = 1e-4) --------
    rnd_info = None
    if not args.no_sweeps:
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        rounded = tt.tt_round(xs, 1e-4)
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        rts = []
        for _ in range(3):
            t = time.perf_counter()
            rounded = tt.tt_round(xs, 1e-4)
            torch.cuda.synchronize(dev)
            rts.append((time.perf_counter() - t) * 1e3)
        rnd_info = {"delta": 1e-4, "ranks_in": list(cfg.r),
                    "ranks_out": [1] + [int(c.shape[2]) for c in rounded],
                    "ms": sorted(rts)[1], "ms_all": rts, "ms_first": (t1 - t0) * 1e3,
                    "note": "synchronous (data-dependent ranks); host wall time, median of 3 "
                            "after one warm-up call (the first includes allocator growth)"}
        # the other row-3 steps at the interior core: left orthonormalisation of the train,
        # the block-index move with the 4-component KKT block index, AMEn enrichment
        def wall(fn, reps=2):
            fn()
            torch.cuda.synchronize(dev)
            t = time.perf_counter()
            for _ in range(reps):
                fn()
            torch.cuda.synchronize(dev)
            return (time.perf_counter() - t) / reps * 1e3
        k = cfg.d // 2
        gen = torch.Generator(device=dev).manual_seed(13)
        rnd = lambda *sh: torch.randn(*sh, dtype=torch.float64, device=dev, generator=gen)
        Wh = rnd(cfg.r[k], cfg.N, 4, cfg.r[k + 1])
        zk = rnd(cfg.r[k], cfg.N, 32)
        rnd_info["orthonormalise_left_ms"] = wall(lambda: tt.tt_orthonormalise(xs, tt.TT_SWEEP_LEFT))
        rnd_info["block_move_right_ms"] = wall(lambda: tt.tt_block_move_right(Wh, xs[k + 1], 1e-6))
        rnd_info["enrich_right_ms"] = wall(lambda: tt.tt_enrich_right(xs[k], zk, xs[k + 1]))
        rnd_info["row3_shapes"] = {"block_move": [cfg.r[k], cfg.N, 4, cfg.r[k + 1]],
                                   "enrich": [cfg.r[k], cfg.N, cfg.r[k + 1], 32]}

    # ---- full sweeps at d = 12 (metric's second half), eager and as a CUDA graph ---------
    sweeps = None
    if not args.no_sweeps:
        sweeps = {}
        # config 5, W5 (tt_sweep_als) without the apply: the timed step's sweep part
        def w5(st):
            tt.tt_sweep_als(xs, As, Xs, Yf, None, phiL, phiR, workspace=ws, stream=st)
        sweeps["config5_W5"] = time_sweep(tt, w5, stream, dev, reps=3)
        # config 4, W34: all right interfaces, all left interfaces, one matvec per core
        inp4 = ttgen.make_inputs(4)
        x4 = [torch.from_numpy(c).to(dev) for c in inp4.x]
        A4 = [torch.from_numpy(c).to(dev) for c in inp4.A]
        pl4 = tt.alloc_interfaces(x4, A4)
        pr4 = tt.alloc_interfaces(x4, A4)
        y4 = [torch.empty_like(c) for c in x4]
        tr4 = tt._Train(x4, A4)
        ws4 = torch.empty(tt.tt_sweep_workspace_size(tr4), dtype=torch.uint8, device=dev)
        wsm4 = torch.empty(max(tt.tt_local_matvec_workspace_size(c.shape[0], c.shape[1], c.shape[2],
                                                                 A.shape[0], A.shape[3], 1)
                               for c, A in zip(x4, A4)), dtype=torch.uint8, device=dev)

        def w34(st):
            tt.tt_sweep_interfaces(x4, A4, pl4, pr4, workspace=ws4, stream=st)
            for k in range(len(x4)):
                tt.tt_local_matvec(pl4[k], A4[k], pr4[k + 1], x4[k], y4[k], workspace=wsm4,
                                   stream=st)
        sweeps["config4_W34_separate_calls"] = time_sweep(tt, w34, stream, dev, reps=20)
        # the same workload as one DAG-scheduled call (matvecs overlap the interface chains)
        ws34 = torch.empty(tt.tt_sweep_w34_workspace_size(tr4), dtype=torch.uint8, device=dev)

        def w34_dag(st):
            tt.tt_sweep_w34(x4, A4, pl4, pr4, y4, workspace=ws34, stream=st)
        sweeps["config4_W34"] = time_sweep(tt, w34_dag, stream, dev, reps=20)
        f34 = bench_w34_flops(ttgen.CONFIGS[4])
        x34 = w34_executed_flops(ttgen.CONFIGS[4])
        sw = sweeps["config4_W34"]
        sw["gflop"] = f34 / 1e9                     # three-stage matvec per core
        sw["executed_gflop"] = x34 / 1e9            # matvecs reuse the left updates' T2_k
        sw["tflops_graph"] = x34 / (sw["graph_ms_median"] * 1e-3) / 1e12
        sw["frac_of_p64"] = sw["tflops_graph"] / p64_sustained
        sw["note"] = ("tflops/frac on executed FLOPs; each matvec is its last stage on the kept "
                      "T2_k of the left update at core k (debug bit 23 restores three stages)")
        # config 3 (d = 10) W34 as well
        inp3 = ttgen.make_inputs(3)
        x3 = [torch.from_numpy(c).to(dev) for c in inp3.x]
        A3 = [torch.from_numpy(c).to(dev) for c in inp3.A]
        pl3, pr3 = tt.alloc_interfaces(x3, A3), tt.alloc_interfaces(x3, A3)
        y3 = [torch.empty_like(c) for c in x3]
        ws3 = torch.empty(tt.tt_sweep_w34_workspace_size(tt._Train(x3, A3)), dtype=torch.uint8,
                          device=dev)

        def w34_c3(st):
            tt.tt_sweep_w34(x3, A3, pl3, pr3, y3, workspace=ws3, stream=st)
        sweeps["config3_W34"] = time_sweep(tt, w34_c3, stream, dev, reps=20)
        sweeps["config3_W34"]["gflop"] = bench_w34_flops(ttgen.CONFIGS[3]) / 1e9
        sweeps["config3_W34"]["executed_gflop"] = w34_executed_flops(ttgen.CONFIGS[3]) / 1e9

    # ---- CPU oracle baseline (rank 0, N=1) ----------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        with pinned_one_core() as pin:
            fl, dt = time_oracle_sample(True)
        cpu = {"value": fl / dt / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": "tt_oracle_local_matvec (1 Krylov column) + tt_oracle_interface_left at "
                         "config-5 interior-core shapes (a=b=256, alpha=beta=36, N=4), "
                         f"{fl / 1e9:.1f} GFLOP in {dt:.1f} s",
               "cpu": cpu_model(), "compiler": "gcc -O2 -std=c99", "pinned_core": pin.core}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"config {cfg.index}: d={cfg.d}, N={cfg.N}, r={max(cfg.r)}, "
                                   f"R={max(cfg.R)}, K={cfg.nvec} Krylov block; W5 two-direction "
                                   "sweep (tt_sweep_als) + full unrounded apply (tt_operator_apply)",
                       "step_gflop": work["step_flops"] / 1e9,
                       "l2": "flushed between timed steps (256 MiB memset outside step events); "
                             "inputs 0.43 GB > L2",
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "clocks": clk,
            "sweeps_d12": sweeps,
            "local_gmres": gm,
            "kkt_block_action": kkt,
            "two_site_matvec": two,
            "tt_round": rnd_info,
            "local_lobpcg": lob,
            "detail": {
                "full_sweep_ms": (total_ms / args.steps) - (apply_detail["ms_per_step"]
                                                            if apply_detail else 0.0),
                "batched_matvec_tflops": mv_tf,
                "batched_matvec_frac_of_p64": mv_tf / p64_sustained,
                "p64_tflops_sustained": p64_sustained, "p64_tflops_burst": p64_burst,
                "apply": apply_detail,
                "stages": stages,
                "step_ms": step_ms,
                "work_gflop": {k: v / 1e9 for k, v in work.items() if k.endswith("flops")},
            },
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
