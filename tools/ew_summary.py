"""Per-launch time / DRAM bytes / GB/s from an ncu --csv launch list with
dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum (dev tool)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
out = {}
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        k = (int(d["ID"]), d["Kernel Name"][:48])
        out.setdefault(k, {})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tsc = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}
print(f"{'id':>3} {'kernel':48} {'us':>8} {'MB':>7} {'GB/s':>6}")
for (i, k), m in sorted(out.items()):
    t, tu = m["gpu__time_duration.sum"]
    rd, ru = m["dram__bytes_read.sum"]
    wr, wu = m["dram__bytes_write.sum"]
    ts = t * tsc[tu]
    b = rd * sc[ru] + wr * sc[wu]
    print(f"{i:3d} {k:48} {ts * 1e6:8.1f} {b / 1e6:7.0f} {b / ts / 1e9:6.0f}")
