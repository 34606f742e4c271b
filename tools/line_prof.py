"""Per-source-line summary of an ncu source page (--print-source cuda,sass --csv)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
cur = None
out = []
hdr = None
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': hdr = r; continue
    if r[0] and r[0] != 'Function Name' and hdr and r[0].isdigit():
        try:
            s = float(r[4]); i = float(r[7])
        except ValueError:
            continue
        out.append((cur, int(r[0]), r[1].strip()[:70], s, i))
ts = sum(o[3] for o in out); ti = sum(o[4] for o in out)
print(f"samples {ts:.0f} instr {ti:.3e}")
for f, ln, src, s, i in sorted(out, key=lambda o: -o[3])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{f:18s}{ln:5d} {100*s/ts:5.1f}% {100*i/ti:5.1f}%  {src}")
