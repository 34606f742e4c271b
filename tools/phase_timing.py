"""Phase breakdown of the v3 kernel (diagnostic build with -DLHAF_PHASE_TIMING): cycles of
thread 0 of each team in decode/build, reduction, (unused), La Budde, series, end barrier.
    python tools/phase_timing.py build        (here: compiles tools/_diag/liblhaf_timing.so)
    python tools/phase_timing.py run [cfg]    (GPU box)"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SO = os.path.join(ROOT, "tools", "_diag", "liblhaf_timing.so")
if sys.argv[1] == "build":
    os.environ["LHAF_NVCC_EXTRA"] = "-DLHAF_PHASE_TIMING"
    from paper_2108_01622_b200 import build as b
    print(b.build(out=SO))
    sys.exit(0)
os.environ["LHAF_LIB_PATH"] = SO
import torch  # noqa
import paper_2108_01622_b200 as L, gbs_inputs as G
lib = ctypes.CDLL(SO)
buf = (ctypes.c_ulonglong * 8)()
for c in [int(x) for x in sys.argv[2:]] or [2, 4, 5]:
    cfg = G.config(c)
    reps = cfg.get('reps_batch', cfg.get('reps'))
    job = L.Job(cfg['A'], cfg['gamma'], reps, mixed=cfg['mixed'])
    U = job.units if c in (1, 2, 3) else max(1, job.units // 64)
    job.reset(); job.run(0, U); torch.cuda.synchronize()
    lib.lhaf_debug_phase_cycles(buf)
    job.reset(); job.run(0, U); torch.cuda.synchronize()
    lib.lhaf_debug_phase_cycles(buf)
    terms = job.terms * U / job.units
    names = ["decode+build", "column: update+carry", "(unused)", "La Budde", "series", "end barrier",
             "column: pivot+publish", "column: barrier wait"]
    tot = sum(buf[i] for i in range(8))
    print(f"cfg{c}: terms={terms:.0f} cycles/term (thread 0 of each team): " +
          ", ".join(f"{nm}={buf[i]/terms:.0f} ({100*buf[i]/tot:.0f}%)" for i, nm in enumerate(names)), flush=True)
    job.close()
