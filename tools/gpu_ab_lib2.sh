# same-box A/B of two libspl builds on the split attention kernels (head_dim 128 / 160):
# per-kernel ncu times at the 175B and 530B (t = 8 simulated) shapes (dev tool)
set +e
for shape in 175B 530B; do
for v in old new old new; do cp ab/libspl_$v.so paper_2205_05198_b200/libspl.so
  AB_SHAPE=$shape timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fa_fwd_umma|fa_bwd_dkdv|fa_bwd_dq_umma" -c 6 --csv python tools/ab_attn.py 2>/dev/null > /tmp/ab.csv
  python - "$shape" "$v" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open('/tmp/ab.csv')) if len(r) > 10]
h = rows[0]; ki = h.index('Kernel Name'); vi = len(h) - 1
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki].split('<')[0].split('(')[0].split()[-1]].append(float(r[vi].replace(',', '')))
print(sys.argv[1], sys.argv[2], {k: round(sum(v) / len(v)) for k, v in d.items()})
PY
done; done
cp ab/libspl_new.so paper_2205_05198_b200/libspl.so
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_widths.py tests/test_gpu_golden.py -q -x -p no:cacheprovider 2>&1 | tail -2
