set +e
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_widths.py tests/test_gpu_golden.py -x -q -p no:cacheprovider > gpurun_out/pp_tests.log 2>&1; echo pytest $?
tail -3 gpurun_out/pp_tests.log
for v in 0 1 0 1; do SPL_ATTN_FWD_PP=$v timeout 300 python tools/ab_attn.py; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fa_fwd|fa_bwd|keep_bits" -c 12 --csv python tools/ab_attn.py 2>/dev/null | grep -E "fa_fwd|fa_bwd|keep" | awk -F'","' '{print $5, $NF}' | cut -c1-150
