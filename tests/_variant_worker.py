"""Worker for tests/test_gpu_variants.py: lhaf_rpt of the seeded cases under the kernel
instantiation chosen by LHAF_V3_ALT (read once per process); prints JSON [[re, im], ...]."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2108_01622_b200 as L  # noqa: E402
import _variant_cases as VC  # noqa: E402

if os.environ.get("LHAF_KERNEL"):
    L.lhaf_set_kernel(int(os.environ["LHAF_KERNEL"]))
res = []
for c in VC.cases():
    v = L.lhaf_rpt(c["A"], c["gamma"], c["reps"])
    res.append([v.real, v.imag])
print(json.dumps(res))
