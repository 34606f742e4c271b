#!/usr/bin/env python3
"""bench.py -- sieve terms/s and seconds per loop hafnian on B200 (BASELINE.json metric).

Workload (default `--workload cfg4`): BASELINE.json config 4, the n = 60 loop hafnian
(Haar m = 100, tanh r = 0.9, gamma sigma = 0.1, 60 photons in 60 distinct modes: d = 60,
2^29 evaluated sieve terms).  One "step" is one pass of the whole hot path (S8(a) a4-a12:
decode, scale, Hessenberg, La Budde, loop terms, series, compensated accumulate, all-reduce,
finalize) over one fixed slice of the lhaf's work units; the lhaf is cut into `--slices`
(default 64, 2^23 terms and 2048 work units per step) contiguous slices; `--steps 64`
evaluates the whole loop hafnian once (then `s_per_lhaf` is measured, not extrapolated).  Other workloads:
cfg2 (the 4096-pattern batch, one step = the whole batch), cfg3 (n = 40 collision-heavy lhaf),
cfg5 (mixed state).

Timing: W untimed warm-up steps; then barrier + cuda synchronize, CUDA events on the launch
stream around exactly K steps, synchronize + barrier; max over ranks.  Between steps a 256 MiB
buffer is written (L2 flush, inside the timed region; ~40 us per step).  nvidia-smi samples
SM clocks and throttle reasons during the timed region.  The e2e number times the public
C-ABI call (lhaf_rpt with host buffers: H2D copies of A/gamma/plan, D2H of the result) for
one whole loop hafnian.  The roofline kernel time is measured with CUDA events around the
sieve launches on the same stream.

Multi-GPU: `--gpus N` without WORLD_SIZE re-launches itself through torchrun (one process per
GPU; fails loudly if fewer than N GPUs are visible); the library's NCCL communicator is
bootstrapped through torch.distributed.  Per step: each rank evaluates its share of the step's
slice, then one ncclAllReduce of that slice's unit partials (exact: disjoint supports).  The
per-rank work per step is fixed (slices = 64 / N for cfg4: weak scaling).

`--impl reference` times the CPU oracle (oracle/, long double, OpenMP) on a bounded sample of
the same workload's terms (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import gbs_inputs as G  # noqa: E402

WORKLOADS = {
    "cfg4": dict(cfg=4, slices=64, desc="BASELINE config 4: single n=60 loop hafnian, m=100 Haar, tanh r=0.9, gamma sigma=0.1, 60 distinct modes, 2^29 evaluated terms at d=60"),
    "cfg2": dict(cfg=2, slices=1, desc="BASELINE config 2: batch of 4096 loop hafnians, N=24 distinct modes of m=50, 2^11 evaluated terms each at d=24"),
    "cfg3": dict(cfg=3, slices=1, desc="BASELINE config 3: n=40 collision-heavy loop hafnian, 16 modes of m=100, gamma=0"),
    "cfg5": dict(cfg=5, slices=128, desc="BASELINE config 5: mixed-state lhaf, 36 photons over 24 modes, eta=0.3, 2k=200, greedy matching of the doubled pattern (DESIGN C11b), d=48"),
    "n40": dict(cfg=40, slices=1, desc="supplementary N=40 collision-free point (SURVEY 8(d)): cfg4 construction with 40 distinct modes, d=40, 2^19 evaluated terms; one step = one whole loop hafnian"),
}
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak.json")


def fp64_peak():
    """Measured FP64 DFMA peak (tools/ubench, committed under profiles/), else spec-derived."""
    try:
        with open(FP64_PEAK_FILE) as f:
            j = json.load(f)
        return float(j["fp64_tflops_sustained"]), "measured DFMA microbenchmark (profiles/fp64_peak.json)"
    except Exception:
        return 148 * 64 * 2 * 1.965e9 / 1e12, "spec-derived 148 SM x 64 DFMA/clk x 2 x 1.965 GHz"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_workload(name):
    w = WORKLOADS[name]
    cfg = G.config(w["cfg"])
    reps = cfg.get("reps_batch", cfg.get("reps"))
    return w, cfg, reps


def run_reference(args, rank):
    """CPU oracle arm: the oracle as it stands, on a bounded sample of the workload's terms."""
    if rank != 0:
        return
    import oracle
    w, cfg, reps = load_workload(args.workload)
    r0 = reps[0] if reps.ndim == 2 else reps
    nthreads = oracle.num_threads()
    per_step = args.ref_terms
    t_total = 0.0
    terms = 0
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        _, c = oracle.fds_range(cfg["A"], cfg["gamma"], r0, s * per_step, (s + 1) * per_step,
                                mixed=cfg["mixed"])
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            t_total += dt
            terms += c
    val = terms / t_total
    line = {
        "impl": "reference", "metric": "sieve terms/s", "value": val, "unit": "terms/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_total / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f80 (x87 long double)", "data": "synthetic",
        "config": {"workload": args.workload, "desc": w["desc"]},
        "cpu_baseline": {"value": val, "unit": "terms/s", "cores": nthreads, "kind": "oracle",
                         "sample": f"{per_step} consecutive sieve terms per step of {args.workload} via oracle.fds_range (explicit long-double powers)"},
        "e2e": {"value": val, "unit": "terms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(cfg, reps, seconds_target=22.0):
    import oracle
    nthreads = oracle.num_threads()
    if reps.ndim == 2:
        # batch workload: whole patterns in order until the time target (each pattern's
        # evaluated terms [0, T_eval) via the oracle's FDS)
        cnt, t0, b = 0, time.perf_counter(), 0
        while b < reps.shape[0] and time.perf_counter() - t0 < seconds_target:
            r = reps[b]
            _, c = oracle.fds_range(cfg["A"], cfg["gamma"], r, 0, 1 << 62, mixed=cfg["mixed"])
            cnt += c
            b += 1
        dt = time.perf_counter() - t0
        return {"value": cnt / dt, "unit": "terms/s", "cores": nthreads, "kind": "oracle",
                "sample": f"{b} whole patterns ({cnt} sieve terms) of the batch via oracle.fds_range, {dt:.1f} s"}
    r0 = reps
    n = max(nthreads, 16)
    t0 = time.perf_counter()
    oracle.fds_range(cfg["A"], cfg["gamma"], r0, 0, n, mixed=cfg["mixed"])
    dt = time.perf_counter() - t0
    n2 = int(max(n, min(200000, n * seconds_target / max(dt, 1e-6))))
    t0 = time.perf_counter()
    _, c = oracle.fds_range(cfg["A"], cfg["gamma"], r0, n, n + n2, mixed=cfg["mixed"])
    dt = time.perf_counter() - t0
    return {"value": c / dt, "unit": "terms/s", "cores": nthreads, "kind": "oracle",
            "sample": f"{c} consecutive sieve terms of the workload's pattern 0 via oracle.fds_range, {dt:.1f} s"}


def slice_bounds(U, s, slices, rank, world):
    """Units of step s: the slice [sb, se) of U work units and this rank's share [ub, ue)."""
    s %= slices
    sb, se = U * s // slices, U * (s + 1) // slices
    return sb, se, sb + (se - sb) * rank // world, sb + (se - sb) * (rank + 1) // world


def hot_path_step(job, s, U, slices, rank, world, stream, out_ptr, between=None):
    """One pass of the hot path over step s's slice: zero the slice's partials, evaluate this
    rank's share (a4-a11), all-reduce the slice (a12; exact, each unit is owned by one rank),
    finalize (a12).  `between(ub, ue)` brackets the evaluation (kernel timing)."""
    sb, se, ub, ue = slice_bounds(U, s, slices, rank, world)
    job.reset_range(sb, se, stream)
    if between:
        between(ub, ue, True)
    job.run(ub, ue, stream)
    if between:
        between(ub, ue, False)
    job.allreduce_range(sb, se, stream)
    job.finalize_dev(out_ptr, stream)


def survey_flops_per_term(d, n):
    """SURVEY 8(d)'s algorithmic work per sieve term (App. A.7): Householder Hessenberg
    (40/3) d^3 + La Budde (4/3) d^3 + loop terms 4 min(n, d) d^2 + Newton 8 n d + series 4 n^2
    real FP64 flops -- the declared model the roofline fraction is quoted against."""
    return (40.0 / 3.0) * d ** 3 + (4.0 / 3.0) * d ** 3 + 4.0 * min(n, d) * d * d + 8.0 * n * d + 4.0 * n * n


def relaunch_with_torchrun(n):
    """bench.py --gpus N without WORLD_SIZE: start N ranks (one per GPU) through torchrun."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"error": f"--gpus {n} requested but only {have} CUDA device(s) are visible"}), flush=True)
        sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")       # NCCL init lines (transport, NVLS) on stderr
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd, env=env))


def time_whole_lhaf(L, cfg_id, reps_override=None, repeats=5):
    """Seconds per loop hafnian of a whole (small) instance through the job API, CUDA events
    around run + finalize on one stream, median of `repeats` after one warm-up."""
    import torch
    c = G.config(cfg_id)
    reps = c["reps"] if reps_override is None else reps_override
    job = L.Job(c["A"], c["gamma"], reps, mixed=c["mixed"])
    st = torch.cuda.current_stream()
    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    times = []
    for r in range(repeats + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        job.reset(st.cuda_stream)
        job.run(0, job.units, st.cuda_stream)
        job.finalize_dev(out.data_ptr(), st.cuda_stream)
        b.record(st)
        torch.cuda.synchronize()
        if r:
            times.append(a.elapsed_time(b) * 1e-3)
    terms = job.terms
    job.close()
    return {"s_per_lhaf": float(np.median(times)), "terms": int(terms), "d": int(job.info.d_max),
            "n": int(job.info.n_max), "terms_per_s": terms / float(np.median(times)), "repeats": repeats}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=sorted(WORKLOADS))
    ap.add_argument("--slices", type=int, default=None)
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-n40", action="store_true")
    ap.add_argument("--ref-terms", type=int, default=256)
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    if args.steps is None:
        args.steps = 5

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch_with_torchrun(args.gpus)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        sys.exit(2)

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"rank {rank}: no CUDA device {local} (visible: {torch.cuda.device_count()})")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2108_01622_b200 as L
    if args.kernel:
        L.lhaf_set_kernel(args.kernel)
    if world > 1:
        uid = [L.lhaf_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        L.lhaf_init_rank(rank, world, uid[0], local)
        print(f"rank {rank}/{world}: library NCCL communicator up on cuda:{local}", file=sys.stderr, flush=True)
    else:
        L.lhaf_set_device(local)

    w, cfg, reps = load_workload(args.workload)
    job = L.Job(cfg["A"], cfg["gamma"], reps, mixed=cfg["mixed"])
    U = job.units
    # A step is one slice of the lhaf's work units.  Per-rank work per step is held fixed as N
    # grows (slices = base / N, each split across the N ranks: weak scaling, >= 2048 units per
    # rank per step for cfg4); single-slice workloads (whole batch / whole lhaf per step) split
    # the same work across the ranks (strong scaling).
    base = args.slices or w["slices"]
    slices = max(1, base // world)
    scaling = "weak" if base >= world and base > 1 else "strong"
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    out_dev = torch.zeros(2 * job.info.batch, dtype=torch.float64, device="cuda")

    kernel_ev = []
    pending = []

    def kernel_events(ub, ue, start):
        if start:
            pending.append(torch.cuda.Event(enable_timing=True))
            pending[-1].record(stream)
        else:
            b = torch.cuda.Event(enable_timing=True)
            b.record(stream)
            kernel_ev.append((pending.pop(), b, ue - ub))

    def step(s, record=False):
        flush.fill_(float(s))
        hot_path_step(job, s, U, slices, rank, world, sp, out_dev.data_ptr(),
                      kernel_events if record else None)

    # warm-up
    job.reset(sp)
    for s in range(args.warmup):
        step(s)
    torch.cuda.synchronize()
    job.reset(sp)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = L.lhaf_launch_count()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for s in range(args.steps):
            step(s, record=True)
        e1.record(stream)
        torch.cuda.synchronize()
    launches = L.lhaf_launch_count() - launches0
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    kernel_ms = sum(a.elapsed_time(b) for a, b, _ in kernel_ev)
    units_timed = sum(n for _, _, n in kernel_ev)
    terms_per_unit = job.terms / U
    my_terms = units_timed * terms_per_unit
    if world > 1:
        t = torch.tensor([ms, kernel_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
        tt = torch.tensor([my_terms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt)
        total_terms = float(tt[0])
    else:
        total_terms = my_terms
    value = total_terms / (ms * 1e-3)
    result = out_dev.cpu().numpy()
    full_cover = args.steps >= slices
    s_per_lhaf = (job.terms / value) if job.info.batch == 1 else None

    # roofline of the hot path's kernels: the evaluation of a slice (job.run) is the dominant
    # launch group (the tree's level kernels, or the per-term sieve kernel of v1/v3/v5), timed
    # with CUDA events on the launch stream.  achieved = the kernels' algorithmic FP64 flops
    # (job.info.flops_per_term_model: the arithmetic the variant's algorithm performs per
    # evaluated term) x the slice's terms / event time, against the
    # measured DFMA peak.  SURVEY 8(d)'s per-term model F (Householder + La Budde per term) is
    # reported next to it as the equivalent throughput of the per-term method: the tree shares
    # the Schur complements of common prefixes, so it needs far fewer flops per term than F.
    d, n = int(job.info.d_max), int(job.info.n_max)
    flops_term = survey_flops_per_term(d, n)
    own_term = job.info.flops_per_term_model
    peak, peak_src = fp64_peak()
    spec_peak = 148 * 64 * 2 * 1.965e9 / 1e12
    own = my_terms * own_term / (kernel_ms * 1e-3) / 1e12 if kernel_ms > 0 else None
    surveyF = my_terms * flops_term / (kernel_ms * 1e-3) / 1e12 if kernel_ms > 0 else None
    roofline = {"bound": "alu", "achieved": own, "peak": peak, "unit": "TFLOP/s",
                "frac": (own / peak) if own else None, "traffic": None,
                "peak_source": peak_src, "peak_spec": spec_peak,
                "frac_of_spec": (own / spec_peak) if own else None,
                "flops_per_term": own_term,
                "flops_model": ("tree (variant 6): complex MACs of the level kernels per evaluated leaf x 8"
                                if job.info.kernel == 6 else "per-term kernel: useful FP64 flops per term"),
                "kernels": "tree_delta_r/tree_pivot_s/tree_bc_k/tree_leaf_r/tree_reduce_k (+ tree_root_k)"
                           if job.info.kernel == 6 else f"sieve (variant {job.info.kernel})",
                "survey_F_per_term": flops_term,
                "survey_F_equivalent_tflops": surveyF,
                "survey_F_equivalent_frac": (surveyF / peak) if surveyF else None,
                "kernel_share_of_step": kernel_ms / ms if ms > 0 else None}
    for fname, key in (("traffic.json", "traffic"), ("ncu_fp64.json", "fp64_pct_ncu")):
        fpath = os.path.join(ROOT, "profiles", fname)
        if os.path.exists(fpath):
            try:
                roofline[key] = json.load(open(fpath)).get(args.workload)
            except Exception:
                pass

    # e2e: the public C-ABI with host buffers, every step: job create (H2D of A, gamma, plan),
    # run over the step's slice, finalize (D2H of the result); the batch: lhaf_rpt_batch
    e2e = None
    if not args.no_e2e:
        # inputs in pinned host memory (torch pin_memory), viewed as numpy for the C-ABI
        A = torch.from_numpy(np.ascontiguousarray(cfg["A"])).pin_memory().numpy()
        gm = torch.from_numpy(np.ascontiguousarray(cfg["gamma"])).pin_memory().numpy()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e2e_terms = 0.0
        t0 = time.perf_counter()
        for s in range(args.steps):
            if reps.ndim == 2:
                v = L.lhaf_rpt_batch(A, gm, reps)
                e2e_terms += job.terms * (rank == 0)
            else:
                jb = L.Job(A, gm, reps, mixed=cfg["mixed"])
                sb, se, ub, ue = slice_bounds(U, s, slices, rank, world)
                jb.run(ub, ue)
                jb.allreduce_range(sb, se)
                v = jb.finalize()
                e2e_terms += (ue - ub) * terms_per_unit
                jb.close()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt, e2e_terms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
            tt2 = t[1:].clone()
            dist.all_reduce(tt2)
            dt, e2e_terms = float(t[0]), float(tt2[0])
        h2d = A.nbytes + gm.nbytes + int(job.info.h2d_plan_bytes)
        d2h = 16 * job.info.batch
        e2e = {"value": e2e_terms / dt, "unit": "terms/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "s_per_step": dt / args.steps,
               "call": "lhaf_rpt_batch" if reps.ndim == 2 else "lhaf_job_create/run/allreduce/finalize (pinned host buffers)",
               "result_first": [complex(np.atleast_1d(v)[0]).real, complex(np.atleast_1d(v)[0]).imag]}

    # the n = 40 point of the BASELINE metric: seconds per whole loop hafnian, measured (one
    # GPU's worth of work; rank 0): the collision-free N = 40 instance (2^19 terms at d = 40)
    # and cfg3 (N = 40 with collisions)
    # mixed state: the kappa-aware matching search of mixed mode 3 (lhaf_rpt_mixed's default) is
    # a per-lhaf setup cost (candidate sample evaluations); the timed slices use mode 1 (the
    # same term structure and cost per term -- every candidate has the same multiplicities)
    search = None
    if rank == 0 and cfg["mixed"] and world == 1:
        t0 = time.perf_counter()
        j1 = L.Job(cfg["A"], cfg["gamma"], reps, mixed=1)
        t1 = time.perf_counter()
        j3 = L.Job(cfg["A"], cfg["gamma"], reps, mixed=3)
        t2 = time.perf_counter()
        search = {"mode3_setup_s": t2 - t1, "mode1_setup_s": t1 - t0,
                  "search_s": (t2 - t1) - (t1 - t0), "candidates": 16, "samples_per_candidate": 8,
                  "matching_eta": list(j3.plan(0).etas())}
        j1.close(); j3.close()
    n40 = None
    if rank == 0 and world == 1 and not args.no_n40 and args.workload == "cfg4":
        try:
            n40 = {"n40_distinct": time_whole_lhaf(L, 40), "cfg3_collisions": time_whole_lhaf(L, 3)}
        except Exception as ex:
            n40 = {"error": str(ex)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline_sample(cfg, reps)
        except Exception as ex:  # the oracle is test infrastructure; never fatal for the bench
            cpu = {"error": str(ex)}

    if rank == 0:
        kappa = None
        if full_cover and job.info.batch == 1:
            kappa = float(job.abs_sum()[0] / max(abs(complex(result[0], result[1])), 1e-300))
        line = {
            "metric": "sieve terms/s", "value": value, "unit": "terms/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.workload, "desc": w["desc"], "slices": slices,
                       "units": U, "terms_per_lhaf": job.terms, "d": d, "n": n,
                       "kernel_variant": job.info.kernel,
                       "l2": "256 MiB buffer written before every step (inside the timed region)",
                       "parallelism": f"term-range shards x{world}"},
            "s_per_lhaf": s_per_lhaf if full_cover else None,
            "s_per_lhaf_extrapolated": None if full_cover else s_per_lhaf,
            "result": [float(result[0]), float(result[1])] if full_cover and job.info.batch == 1 else None,
            "accuracy": {"kappa": kappa,
                         "pin": "tests/test_gpu_fullsize.py::test_block_diagonal_N60 (P10, P:510; the same default path at d = 60)"},
            "n40": n40,
            "matching_search": search,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    job.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
