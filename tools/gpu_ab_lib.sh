# same-box A/B of two builds of libspl (ab/libspl_old.so vs ab/libspl_new.so): forward / backward
# attention kernel times under ncu and the layer step (dev tool)
set +e
K=${K:-fa_fwd_pp}
for v in old new old new; do cp ab/libspl_$v.so paper_2205_05198_b200/libspl.so
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$K -c 3 --csv python tools/ab_attn.py 2>/dev/null | grep $K | awk -F'","' -v v=$v '{print "ncu " v, $NF}'; done
cp ab/libspl_new.so paper_2205_05198_b200/libspl.so
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_widths.py tests/test_gpu_golden.py -q -x -p no:cacheprovider 2>&1 | tail -2
