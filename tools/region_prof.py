"""Aggregate an ncu source page (--print-source cuda,sass --csv) by function of lhaf_v3.cu:
samples (stall-weighted time) and executed instructions per region."""
import csv, re, sys, os
SRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2108_01622_b200", "csrc", "lhaf_v3.cu")
lines = open(SRC).read().split("\n")
starts = []
for i, l in enumerate(lines, 1):
    m = re.match(r"^(?:__device__|__global__|sieve_v3|terms_v3).*?(\w+)\(", l)
    if m:
        starts.append((i, m.group(1)))
def region(ln):
    name = "?"
    for s, n in starts:
        if s <= ln: name = n
    return name
rows = list(csv.reader(open(sys.argv[1])))
cur = None; hdr = None; agg = {}; ts = ti = 0
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr and r[0].isdigit():
        try: s = float(r[4]); i = float(r[7])
        except ValueError: continue
        name = region(int(r[0])) if cur == "lhaf_v3.cu" else "[" + cur + "]"
        a = agg.setdefault(name, [0, 0]); a[0] += s; a[1] += i; ts += s; ti += i
for k, (s, i) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:28s} samples {100*s/ts:5.1f}%  instr {100*i/ti:5.1f}%")
