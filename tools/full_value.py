"""One complete loop hafnian of a BASELINE config (every evaluated term), for the accuracy study
of DESIGN.md section 6: value, kappa = sum|term| / |lhaf|, wall time.  Appends a JSON line to
gpurun_out/full_values.jsonl.

python tools/full_value.py CFG PREC PERM [MIXEDMODE]
  PREC 0/1 (lhaf_set_precision), PERM -1 = the config as generated, else a seeded permutation of
  the modes (a different matching / term order / rounding of the same lhaf), MIXEDMODE 1 =
  greedy doubled pattern, 2 = natural pairing (mixed configs; default: the mode's own choice)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import gbs_inputs as G
import paper_2108_01622_b200 as L

cfg_id, prec, perm = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
mixed_mode = int(sys.argv[4]) if len(sys.argv) > 4 else 1
kernel = int(os.environ.get("LHAF_KERNEL", "0"))
cfg = G.config(cfg_id)
A, g, reps = cfg["A"], cfg["gamma"], cfg["reps"]
if perm >= 0:
    k = reps.shape[0]
    P = np.random.default_rng(perm).permutation(k)
    if cfg["mixed"]:
        P2 = np.concatenate([P, P + k])
        A, g = A[np.ix_(P2, P2)], g[P2]
    else:
        A, g = A[np.ix_(P, P)], g[P]
    reps = reps[P]
L.lhaf_set_precision(prec)
if kernel:
    L.lhaf_set_kernel(kernel)
t0 = time.time()
job = L.Job(A, g, reps, mixed=mixed_mode if cfg["mixed"] else 0)
job.reset(); job.run(); v = job.finalize()[0]
kappa = job.abs_sum()[0] / abs(v)
dt = time.time() - t0
rec = dict(cfg=cfg_id, prec=prec, perm=perm, mixed_mode=mixed_mode if cfg["mixed"] else None,
           kernel=int(job.info.kernel), terms=int(job.terms), re=v.real, im=v.imag, kappa=kappa,
           seconds=dt, terms_per_s=job.terms / dt)
job.close()
print(json.dumps(rec), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "full_values.jsonl"), "a") as f:
    f.write(json.dumps(rec) + "\n")
