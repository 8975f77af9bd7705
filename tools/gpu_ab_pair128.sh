set +e
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_layer.py tests/test_gpu_widths.py tests/test_gpu_fused_ag.py tests/test_gpu_ipc.py -x -q -p no:cacheprovider 2>&1 | tail -2
for v in 0 1 0 1; do echo "PAIR128=$v"; SPL_GEMM_PAIR128=$v timeout 300 python tools/layer_times.py --t 8 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin)
for r in d['rows']: print(' ', r['experiment'], round(r['combined_ms'],3))"; done
