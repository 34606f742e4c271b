"""Quick device-side throughput check of the sieve kernel on the five configs (slices for 4/5)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2108_01622_b200 as L, gbs_inputs as G
if len(sys.argv) > 1: L.lhaf_set_kernel(int(sys.argv[1]))
st = torch.cuda.current_stream().cuda_stream
for c in [1, 2, 3, 4, 5]:
    cfg = G.config(c)
    reps = cfg.get('reps_batch', cfg.get('reps'))
    job = L.Job(cfg['A'], cfg['gamma'], reps, mixed=cfg['mixed'])
    U = job.units
    frac_units = U if c in (1, 2, 3) else max(1, U // 64)
    terms = job.terms * frac_units / U
    job.reset(st); job.run(0, frac_units, st); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); job.run(0, frac_units, st); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    fl = job.info.flops_per_term_model
    print(f"cfg{c}: d={job.info.d_max} n={job.info.n_max} units={frac_units}/{U} terms={terms:.3e} "
          f"ms={ms:.2f} terms/s={terms/ms*1e3:.3e} model_flops/term={fl:.3e} TF/s={terms*fl/ms/1e9:.2f}", flush=True)
    job.close()
