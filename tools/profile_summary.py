"""Summarise an ncu launch list with gpu__time_duration + dram bytes (dev tool).
usage: python tools_profile_summary.py <launches.csv> <out.json>"""
import csv
import json
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr, recs = None, defaultdict(dict)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        recs[d["ID"]]["name"] = d["Kernel Name"]
        recs[d["ID"]][d["Metric Name"]] = float(d["Metric Value"])
fam = defaultdict(lambda: dict(n=0, ns=0.0, rd=0.0, wr=0.0))
for v in recs.values():
    m = re.search(r"(fa_\w+|gemm_tc\w*<[^>]*>|keep_bits_k|ln_\w+|bdr_\w+<[^>]*>|dropout\w+|colsum\w+|reduce\w+|rs_local_k|\w+_k)", v["name"])
    key = m.group(1) if m else v["name"][:60]
    f = fam[key]
    f["n"] += 1
    f["ns"] += v.get("gpu__time_duration.sum", 0)
    f["rd"] += v.get("dram__bytes_read.sum", 0)
    f["wr"] += v.get("dram__bytes_write.sum", 0)
tot = sum(f["ns"] for f in fam.values())
out = {}
print(f"{'kernel':60s} {'n':>3} {'ms/launch':>10} {'share':>6} {'DRAM MB/launch':>15} {'GB/s':>8}")
for k, f in sorted(fam.items(), key=lambda x: -x[1]["ns"]):
    ms = f["ns"] / f["n"] / 1e6
    mb = (f["rd"] + f["wr"]) / f["n"] / 1e6
    gbs = (f["rd"] + f["wr"]) / f["ns"] if f["ns"] else 0
    out[k] = dict(launches=f["n"], ms_per_launch=ms, share=f["ns"] / tot,
                  dram_read_bytes_per_launch=f["rd"] / f["n"], dram_write_bytes_per_launch=f["wr"] / f["n"])
    print(f"{k[:60]:60s} {f['n']:3d} {ms:10.3f} {f['ns'] / tot:6.1%} {mb:15.1f} {gbs:8.0f}")
json.dump(out, open(sys.argv[2], "w"), indent=1)
