# same-box A/B of an opt-in GEMM switch: VAR=SPL_GEMM_KSNAKE bash tools/gpu_ab_ks.sh
set +e
V=${VAR:-SPL_GEMM_KSNAKE}
b() { env $V=$2 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('$1', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:(round(v['ms_per_step'],2) if v else None) for k,v in d['rooflines'].items()})"; }
for i in 1 2; do b off 0; b on 1; done
for x in 0 1; do env $V=$x timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tc -c 12 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null > gpurun_out/ab$x.csv; done
env $V=1 timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_widths.py -q -x 2>&1 | tail -3
