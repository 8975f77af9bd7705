set +e
b() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('$1', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:(round(v['ms_per_step'],2) if v else None) for k,v in d['rooflines'].items()})"; }
b base
SPL_KEEPBITS_SIDE=1 b side1024
SPL_KEEPBITS_SIDE=1 SPL_KEEPBITS_NT=512 b side512
SPL_KEEPBITS_SIDE=1 SPL_KEEPBITS_NT=384 b side384
b base
SPL_KEEPBITS_SIDE=1 SPL_KEEPBITS_NT=512 b side512
