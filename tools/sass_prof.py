"""Summarise an ncu source-page CSV (--page source --csv --print-source sass): samples and
executed instructions per opcode, and the hottest instructions with their stall columns."""
import csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
col = {h: i for i, h in enumerate(hdr)}
def num(x):
    try: return float(x)
    except: return 0.0
tot_s = sum(num(r[col['Warp Stall Sampling (All Samples)']]) for r in data)
tot_i = sum(num(r[col['Instructions Executed']]) for r in data)
ops = {}
for r in data:
    src = r[col['Source']]
    m = re.match(r'\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)', src)
    op = m.group(2) if m else '?'
    o = ops.setdefault(op, [0, 0])
    o[0] += num(r[col['Warp Stall Sampling (All Samples)']]); o[1] += num(r[col['Instructions Executed']])
print(f"total samples {tot_s:.0f}  instructions {tot_i:.3e}")
for op, (s, i) in sorted(ops.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{op:10s} samples {100*s/tot_s:5.1f}%  instr {100*i/tot_i:5.1f}%")
stall_cols = [h for h in hdr if h.startswith('stall_')]
print("stall totals:")
st = {h: sum(num(r[col[h]]) for r in data) for h in stall_cols}
for h, v in sorted(st.items(), key=lambda x: -x[1])[:12]:
    print(f"  {h:30s} {100*v/max(tot_s,1):5.1f}%")
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print("hottest:")
for r in sorted(data, key=lambda r: -num(r[col['Warp Stall Sampling (All Samples)']]))[:N]:
    top = sorted(((h, num(r[col[h]])) for h in stall_cols), key=lambda x: -x[1])[:3]
    print(f"{r[col['Address']]:>6s} {num(r[col['Warp Stall Sampling (All Samples)']]):6.0f} {r[col['Source']][:60]:60s} {top}")
