"""Diagnostic: cycles per term in the v5 reduction vs the tail (La Budde + series), from a
-DLHAF_V5_TIMING build of the library at tools/_diag/liblhaf_v5t.so.  python tools/v5_phase.py build|run"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tools", "_diag", "liblhaf_v5t.so")
if sys.argv[1] == "build":
    os.environ["LHAF_NVCC_EXTRA"] = "-DLHAF_V5_TIMING"
    from paper_2108_01622_b200 import build as b
    b.build(out=OUT)
    sys.exit(0)
os.environ["LHAF_LIB_PATH"] = OUT
import numpy as np, gbs_inputs as G
import paper_2108_01622_b200 as L
lib = ctypes.CDLL(OUT)
buf = (ctypes.c_ulonglong * 4)()
for c, slices in ((4, 64), (5, 128), (40, 1)):
    cfg = G.config(c)
    job = L.Job(cfg["A"], cfg["gamma"], cfg["reps"], mixed=cfg["mixed"])
    ue = max(1, job.units // slices)
    lib.lhaf_debug_v5_phase(buf)
    job.reset(); job.run(0, ue)
    lib.lhaf_debug_v5_phase(buf)
    n = buf[2]
    print(f"cfg{c} kernel {job.info.kernel}: terms {n}, cycles/term reduce {buf[0]/n:.0f} tail {buf[1]/n:.0f} (La Budde {(buf[3] & 0xffffffffffffffff)/n:.0f})", flush=True)
    job.close()
