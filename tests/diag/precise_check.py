"""GPU check of the precise mode (double-double La Budde + series): per-term errors vs the
long-double oracle (fast vs precise), block-diagonal sums, and the cost on cfg slices."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import gbs_inputs as G
import oracle as O
import paper_2108_01622_b200 as L
import torch

rel = lambda a, b: abs(a - b) / abs(b)
for c, mixed, natural in ((4, False, False), (5, True, True), (5, True, False)):
    cfg = G.config(c)
    if mixed and not natural:
        reps_o, mm = np.concatenate([cfg["reps"], cfg["reps"]]), False
    else:
        reps_o, mm = cfg["reps"], mixed
    C, v, eta, n = O.reduced_system(cfg["A"], cfg["gamma"], reps_o, mixed=mm)
    ts = G.rng_for(99).integers(0, int(np.prod([e + 1 for e in eta])) // 2, 256, dtype=np.uint64)
    W = np.array([O.decode(int(t), eta)[1] for t in ts], np.int32)
    refs = O.fds_terms(C, v, W, n)
    for prec in (0, 1):
        L.lhaf_set_precision(prec)
        job = L.Job(cfg["A"], cfg["gamma"], cfg["reps"], mixed=(2 if natural else 1) if mixed else 0)
        gg = job.terms_g(ts)
        k = job.info.kernel
        job.close()
        e = np.abs(gg - refs) / np.abs(refs)
        print(f"cfg{c}{' natural' if natural else (' greedy' if mixed else '')} prec={prec} kernel {k}: per-term rel err median {np.median(e):.2e} p90 {np.quantile(e, 0.9):.2e} max {e.max():.2e}", flush=True)
L.lhaf_set_precision(0)
for m, seed in ((24, 4801), (20, 4001)):
    rng = G.rng_for(seed)
    A1 = G.random_symmetric(m, rng, 0.5); A2 = G.random_symmetric(m, rng, 0.5)
    g1 = G.complex_gaussian(m, 0.5, rng); g2 = G.complex_gaussian(m, 0.5, rng)
    Z = np.zeros((m, m), complex)
    A = np.block([[A1, Z], [Z, A2]]); g = np.concatenate([g1, g2]); perm = rng.permutation(2 * m)
    want = O.lhaf(A1, g1, [1] * m, method="et") * O.lhaf(A2, g2, [1] * m, method="et")
    for prec in (0, 1):
        L.lhaf_set_precision(prec)
        got = L.lhaf_rpt(A[np.ix_(perm, perm)], g[perm], np.ones(2 * m, np.int32))
        print(f"block-diag N={2*m} prec={prec}: rel err {rel(got, want):.2e}", flush=True)
L.lhaf_set_precision(0)
st = torch.cuda.current_stream()
for c, slices in ((4, 64), (5, 128), (40, 1), (2, 1)):
    cfg = G.config(c)
    reps = cfg.get("reps_batch", cfg.get("reps"))
    for prec in (0, 1):
        L.lhaf_set_precision(prec)
        job = L.Job(cfg["A"], cfg["gamma"], reps, mixed=cfg["mixed"])
        U = job.units
        ue = max(1, U // slices)
        job.reset(); job.run(0, ue); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); job.run(0, ue, st.cuda_stream); b.record(st); torch.cuda.synchronize()
        dt = a.elapsed_time(b) * 1e-3
        print(f"cfg{c} prec={prec} kernel {job.info.kernel}: {ue * job.terms / U / dt:.3e} terms/s", flush=True)
        job.close()
L.lhaf_set_precision(0)
