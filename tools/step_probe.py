"""Per-step timeline of the reduction (diagnostic build with -DLHAF_STEP_PROBE): cycles between
the probes of every warp leader of block 0, averaged over the steps of phase 1 and of the whole
reduction.  python tools/step_probe.py build | run [cfg] [ctas_per_sm]"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SO = os.path.join(ROOT, "tools", "_diag", "liblhaf_probe.so")
if sys.argv[1] == "build":
    os.environ["LHAF_NVCC_EXTRA"] = "-DLHAF_STEP_PROBE"
    from paper_2108_01622_b200 import build as b
    print(b.build(out=SO))
    sys.exit(0)
os.environ["LHAF_LIB_PATH"] = SO
if len(sys.argv) > 3:
    os.environ["LHAF_CTAS_PER_SM"] = sys.argv[3]
import numpy as np  # noqa: E402
import paper_2108_01622_b200 as L, gbs_inputs as G  # noqa: E402
lib = ctypes.CDLL(SO)
c = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = G.config(c)
job = L.Job(cfg["A"], cfg["gamma"], cfg.get("reps_batch", cfg.get("reps")), mixed=cfg["mixed"])
job.reset(); job.run(0, 296)
buf = np.zeros((64, 8, 4), np.int64)
lib.lhaf_debug_step_probe(buf.ctypes.data_as(ctypes.c_void_p))
names = ["top->redux", "redux->publish done", "barrier wait", "keys->m", "slot loop", "shfl+carry", "->next top"]
E = job.info.d_max + 1
steps = [k for k in range(min(E - 2, 63)) if buf[k, 0, 0] and buf[k + 1, 0, 0]]
for label, ks in (("all steps", steps), ("phase 1 (k<12)", [k for k in steps if k < 12]), ("last phase (k>=44)", [k for k in steps if k >= 44])):
    if not ks:
        continue
    d = np.zeros((7, 4))
    for k in ks:
        t = buf[k].astype(float)
        nxt = buf[k + 1, 0].astype(float)
        for i in range(6):
            d[i] += t[i + 1] - t[i]
        d[6] += nxt - t[6]
    d /= len(ks)
    print(f"{label}: {len(ks)} steps, cycles per step (warp leaders 0..3)")
    for i, nm in enumerate(names):
        print(f"  {nm:22s} " + " ".join(f"{x:8.0f}" for x in d[i]))
    print(f"  {'total':22s} " + " ".join(f"{x:8.0f}" for x in d.sum(0)))
