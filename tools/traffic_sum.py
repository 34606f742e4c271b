"""Sum DRAM bytes and time per kernel from an ncu --csv metrics log of a job.run
(dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum); prints JSON.
usage: python tools/traffic_sum.py <ncu.csv> <terms> <label>"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
terms = float(sys.argv[2])
hdr = None
per = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
         "msecond": 1e-3, "second": 1}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1)
        per[k][d["Metric Name"]] += v
        if d["Metric Name"] == "gpu__time_duration.sum":
            cnt[k] += 1
tot_r = sum(p["dram__bytes_read.sum"] for p in per.values())
tot_w = sum(p["dram__bytes_write.sum"] for p in per.values())
tot_t = sum(p["gpu__time_duration.sum"] for p in per.values())
out = {"label": sys.argv[3], "terms": terms, "dram_read_bytes": tot_r, "dram_write_bytes": tot_w,
       "bytes_per_term": (tot_r + tot_w) / terms, "kernel_time_s": tot_t,
       "kernels": {k: {"launches": cnt[k], "time_s": p["gpu__time_duration.sum"],
                       "share": (p["gpu__time_duration.sum"] / tot_t) if tot_t else None,
                       "dram_bytes": p["dram__bytes_read.sum"] + p["dram__bytes_write.sum"]}
                   for k, p in sorted(per.items(), key=lambda x: -x[1]["gpu__time_duration.sum"])}}
print(json.dumps(out, indent=1))
