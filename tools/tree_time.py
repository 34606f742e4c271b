"""Time job.run over a slice of a BASELINE workload for a kernel variant (CUDA events).
usage: python tools/tree_time.py <cfg> <variant> [slices] [reps]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gbs_inputs as G  # noqa: E402
import paper_2108_01622_b200 as L  # noqa: E402

cfgn, var = int(sys.argv[1]), int(sys.argv[2])
slices = int(sys.argv[3]) if len(sys.argv) > 3 else 1
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
L.lhaf_set_kernel(var)
c = G.config(cfgn)
r = c["reps"] if "reps" in c else c["reps_batch"]
t0 = time.time()
job = L.Job(c["A"], c["gamma"], r, mixed=c["mixed"])
U = job.units
st = torch.cuda.current_stream()
ue = max(1, U // slices)
for i in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    job.reset(st.cuda_stream)
    a.record(st)
    job.run(0, ue, st.cuda_stream)
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    terms = job.terms * ue / U
    print(f"cfg{cfgn} variant {job.info.kernel} units {ue}/{U}: {ms:.1f} ms, {terms / ms * 1e3:.4g} terms/s, "
          f"model {job.info.flops_per_term_model:.4g} flop/term -> {terms * job.info.flops_per_term_model / ms * 1e-9:.2f} TFLOP/s", flush=True)
if slices == 1:
    print("value", job.finalize()[0], "abs", job.abs_sum()[0])
