"""Summarise an ncu --page raw --csv export of ONE kernel launch into JSON: duration, FP64 pipe
activity, executed FP64 flops as a fraction of the chip's DFMA peak (2 DFMA + DADD + DMUL thread
instructions per cycle over 148 SM x 64 DFMA/clk x 2), issue activity, occupancy, DRAM traffic,
registers and the top stall reasons.
    python tools/ncu_summary.py RAW.csv [label]"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
data = rows[2:]


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def get(row, name, default=None, scaled=False):
    try:
        i = hdr.index(name)
        v = float(row[i].replace(",", ""))
        return v * SCALE.get(units[i], 1.0) if scaled else v
    except (ValueError, IndexError):
        return default


out = []
for r in data:
    kname = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    dfma = get(r, "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed", 0.0)
    dadd = get(r, "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed", 0.0)
    dmul = get(r, "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed", 0.0)
    peak = get(r, "sm__ops_path_tensor_src_fp64.sum.peak_sustained", 18944.0) or 18944.0
    stalls = {h.split("warps_issue_stalled_")[1].split("_per_issue")[0]: get(r, h)
              for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")}
    top = sorted(((k, v) for k, v in stalls.items() if v and k not in ("selected",)), key=lambda x: -x[1])[:6]
    out.append({
        "label": sys.argv[2] if len(sys.argv) > 2 else None,
        "kernel": kname[:120],
        "duration_ms": get(r, "gpu__time_duration.sum", scaled=True),
        "registers_per_thread": get(r, "launch__registers_per_thread"),
        "grid": get(r, "launch__grid_size"),
        "block": get(r, "launch__block_size"),
        "warps_active_pct": get(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": get(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "fp64_pipe_active_pct": get(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "fp64_executed_flops_per_cycle": 2 * dfma + dadd + dmul,
        "fp64_pct_ncu": (2 * dfma + dadd + dmul) / peak,
        "dram_read_bytes": get(r, "dram__bytes_read.sum", scaled=True),
        "dram_write_bytes": get(r, "dram__bytes_write.sum", scaled=True),
        "top_stalls_per_issue": top,
        "threads_per_inst": {h: get(r, h) for h in hdr if "per_inst_executed" in h},
        "occupancy_limits": {h: get(r, h) for h in hdr if h.startswith("launch__occupancy_limit")},
        "smem_dynamic_bytes": get(r, "launch__shared_mem_per_block_dynamic", scaled=True),
        "inst_executed": get(r, "smsp__inst_executed.sum"),
        "shared_bank_conflicts": {h: get(r, h) for h in hdr if "bank_conflicts" in h and "shared" in h},
    })
print(json.dumps(out if len(out) > 1 else out[0], indent=1))
