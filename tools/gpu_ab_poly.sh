# same-box A/B of the FMA-pipe exponential offload in the ping-pong forward (SPL_ATTN_POLY)
set +e
for pe in 0 4 2 8 0 4 2 8; do echo "pe=$pe $(SPL_ATTN_POLY=$pe timeout 300 python tools/ab_attn.py 2>&1 | tail -1)"; done
for pe in 0 4 0 4; do SPL_ATTN_POLY=$pe timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('bench pe=$pe', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:(round(v['ms_per_step'],3) if v else None) for k,v in d['rooflines'].items()})"; done
for pe in 0 4 2; do SPL_ATTN_POLY=$pe timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fa_fwd_pp -c 3 --csv python tools/ab_attn.py 2>/dev/null | grep fa_fwd_pp | awk -F'","' -v pe=$pe '{print "ncu pe=" pe, $NF}'; done
SPL_ATTN_POLY=4 timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_widths.py tests/test_gpu_golden.py -q -x -p no:cacheprovider 2>&1 | tail -3
