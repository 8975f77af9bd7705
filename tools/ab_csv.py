"""Per-kernel time and DRAM bytes from two ncu --csv launch lists (gpurun_out/ab0.csv, ab1.csv)."""
import csv
import sys

for f in sys.argv[1:]:
    hdr, recs = None, {}
    for r in csv.reader(open(f)):
        if 'Kernel Name' in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            recs.setdefault(d['ID'], {'name': d['Kernel Name']})[d['Metric Name']] = float(d['Metric Value'])
    tb = sum(v.get('dram__bytes_read.sum', 0) + v.get('dram__bytes_write.sum', 0) for v in recs.values())
    tt = sum(v.get('gpu__time_duration.sum', 0) for v in recs.values())
    print(f, len(recs), 'launches', round(tb / max(1, len(recs)) / 1e9, 3), 'GB/launch', round(tt / 1e6, 3), 'ms total')
    for v in recs.values():
        print('   ', round(v.get('gpu__time_duration.sum', 0) / 1e3, 1), 'us',
              round((v.get('dram__bytes_read.sum', 0) + v.get('dram__bytes_write.sum', 0)) / 1e9, 2), 'GB', v['name'][:40])
