"""Summarise an ncu --metrics gpu__time_duration.sum launch list by kernel (dev tool)."""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr, out = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((d["Kernel Name"], float(d["Metric Value"])))
agg = defaultdict(lambda: [0.0, 0])
for k, v in out:
    m = re.search(r"(fa_\w+|gemm_tc_kernel|gemm_simt_k|ln_\w+|bdr_k|dropout\w+|colsum\w+|reduce\w+|rs_local_k|\w+_k)\b", k)
    key = m.group(1) if m else k[:50]
    if key == "gemm_tc_kernel":
        t = re.search(r"gemm_tc_kernel<(\d+), (\w+), (\w+), (\d+)>", k)
        key += f"<BN={t.group(1)},A_MN={t.group(2)},B_MN={t.group(3)},EPI={t.group(4)}>" if t else ""
    agg[key][0] += v
    agg[key][1] += 1
unit = 1e6 if max(v for _, v in out) > 1e4 else 1e3  # ns or us
tot = sum(v for _, v in out)
print(f"{'ms':>9} {'%':>6} {'n':>4}  kernel")
for k, (v, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{v / unit:9.3f} {100 * v / tot:6.1f} {n:4d}  {k}")
print(f"{tot / unit:9.3f}  total over {len(out)} launches")
