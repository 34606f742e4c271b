"""Quick GPU check of a kernel variant against v3 and the oracle, and a timing of a cfg slice.
python tests/diag/v5_check.py [variant=5]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import gbs_inputs as G
import oracle as O
import paper_2108_01622_b200 as L
import torch

var = int(sys.argv[1]) if len(sys.argv) > 1 else 5
rel = lambda a, b: abs(a - b) / abs(b)
# 1) block-diagonal cases (Fig. 5 protocol) at N = 48/40/34 and small random ones
for m, seed in ((24, 4801), (20, 4001), (17, 3401)):
    rng = G.rng_for(seed)
    A1 = G.random_symmetric(m, rng, 0.5); A2 = G.random_symmetric(m, rng, 0.5)
    g1 = G.complex_gaussian(m, 0.5, rng); g2 = G.complex_gaussian(m, 0.5, rng)
    Z = np.zeros((m, m), complex)
    A = np.block([[A1, Z], [Z, A2]]); g = np.concatenate([g1, g2]); perm = rng.permutation(2 * m)
    one = np.ones(2 * m, np.int32)
    want = O.lhaf(A1, g1, [1] * m, method="et") * O.lhaf(A2, g2, [1] * m, method="et")
    for v in (3, var):
        L.lhaf_set_kernel(v)
        got = L.lhaf_rpt(A[np.ix_(perm, perm)], g[perm], one)
        print(f"N={2*m} kernel {v}: rel err {rel(got, want):.2e}", flush=True)
    for gz in (True,):
        L.lhaf_set_kernel(var)
        got = L.lhaf_rpt(A[np.ix_(perm, perm)], np.zeros(2 * m), one)
        L.lhaf_set_kernel(3)
        ref = L.lhaf_rpt(A[np.ix_(perm, perm)], np.zeros(2 * m), one)
        print(f"  no loops: v{var} {got:.6e} v3 {ref:.6e}", flush=True)
L.lhaf_set_kernel(0)
# 2) per-term vs oracle at cfg4 / cfg5
for c, mixed in ((4, False), (5, True)):
    cfg = G.config(c)
    reps_o = np.concatenate([cfg["reps"], cfg["reps"]]) if mixed else cfg["reps"]
    C, v, eta, n = O.reduced_system(cfg["A"], cfg["gamma"], reps_o, mixed=False)
    L.lhaf_set_kernel(var)
    job = L.Job(cfg["A"], cfg["gamma"], cfg["reps"], mixed=mixed)
    info = L.lhaf_plan(cfg["reps"], mixed=mixed)
    ts = G.rng_for(99).integers(0, info.T_eval, 64, dtype=np.uint64)
    gg = job.terms_g(ts)
    print("kernel in job:", job.info.kernel)
    job.close()
    W = np.array([O.decode(int(t), eta)[1] for t in ts], np.int32)
    refs = O.fds_terms(C, v, W, n)
    e = np.abs(gg - refs) / np.abs(refs).max()
    print(f"cfg{c} per-term: max {e.max():.2e} median {np.median(e):.2e}", flush=True)
# 3) timing: a slice of cfg4 / cfg5 with both kernels
st = torch.cuda.current_stream()
for c, slices in ((4, 64), (5, 128), (40, 1)):
    cfg = G.config(c)
    for v in (3, var):
        L.lhaf_set_kernel(v)
        job = L.Job(cfg["A"], cfg["gamma"], cfg["reps"], mixed=cfg["mixed"])
        U = job.units
        ue = max(1, U // slices)
        job.reset(); job.run(0, ue); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        job.run(0, ue, st.cuda_stream)
        b.record(st)
        torch.cuda.synchronize()
        dt = a.elapsed_time(b) * 1e-3
        print(f"cfg{c} kernel {job.info.kernel}: {ue * job.terms / U / dt:.3e} terms/s ({dt:.3f} s)", flush=True)
        job.close()
L.lhaf_set_kernel(0)
