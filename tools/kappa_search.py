"""kappa = sum|term| / |lhaf| of a pattern under different pair matchings (the greedy matching
of the pattern with its modes permuted): estimated from sampled terms (job.terms_g, times the
binomial weight from lhaf_decode) and, for a few matchings, exact from a full evaluation.
    python tools/kappa_search.py CFG [NPERM] [SAMPLES] [FULL]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gbs_inputs as G
import paper_2108_01622_b200 as L

cfg_id = int(sys.argv[1]); nperm = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ns = int(sys.argv[3]) if len(sys.argv) > 3 else 4096; nfull = int(sys.argv[4]) if len(sys.argv) > 4 else 2
cfg = G.config(cfg_id)
out = []
for perm in range(-1, nperm):
    A, g, reps = cfg["A"], cfg["gamma"], cfg["reps"]
    if perm >= 0:
        k = reps.shape[0]
        P = np.random.default_rng(perm).permutation(k)
        if cfg["mixed"]:
            P2 = np.concatenate([P, P + k]); A, g = A[np.ix_(P2, P2)], g[P2]
        else:
            A, g = A[np.ix_(P, P)], g[P]
        reps = reps[P]
    job = L.Job(A, g, reps, mixed=1 if cfg["mixed"] else 0)
    info = job.plan(0)
    rng = np.random.default_rng(99)
    ts = rng.integers(0, info.T_eval, ns, dtype=np.uint64)
    t0 = time.time()
    gv = job.terms_g(ts)
    wts = np.array([L.lhaf_decode(info, int(t))[3] for t in ts], float)
    est = info.T_eval * np.mean(np.abs(gv) * wts) * 2.0 ** (1 - info.n)
    rec = dict(perm=perm, H=info.H, T_eval=int(info.T_eval), etas=info.etas(), est_abs_sum=est,
               sample_s=time.time() - t0)
    if perm < nfull - 1:
        job.reset(); job.run(); v = job.finalize()[0]
        rec.update(value=[v.real, v.imag], abs_sum=job.abs_sum()[0], kappa=job.abs_sum()[0] / abs(v))
    job.close()
    out.append(rec)
    print(json.dumps(rec), flush=True)
