set +e
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fa_bwd_fused|fa_fwd" -c 4 --csv python tools/ab_attn.py 2>/dev/null | grep -E "fa_" | awk -F'","' '{print $5, $NF}' | cut -c1-140
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_golden.py tests/test_gpu_widths.py -x -q -p no:cacheprovider 2>&1 | tail -2
