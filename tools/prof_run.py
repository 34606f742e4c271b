"""One sieve launch over a unit range of a config (for ncu --set full captures)."""
import sys, torch
sys.path.insert(0, '.')
import paper_2108_01622_b200 as L, gbs_inputs as G
cfg_id = int(sys.argv[1]); frac = int(sys.argv[2]) if len(sys.argv) > 2 else 1
if len(sys.argv) > 3: L.lhaf_set_kernel(int(sys.argv[3]))
cfg = G.config(cfg_id)
reps = cfg.get('reps_batch', cfg.get('reps'))
job = L.Job(cfg['A'], cfg['gamma'], reps, mixed=cfg['mixed'])
U = max(1, job.units // frac) if frac > 0 else min(job.units, -frac)
st = torch.cuda.current_stream().cuda_stream
job.reset(st); job.run(0, U, st); torch.cuda.synchronize()
print("units", U, "of", job.units, "terms", job.terms * U // job.units, "flops/term", job.info.flops_per_term_model)
