set +e
b() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('$1', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:(round(v['ms_per_step'],2) if v else None) for k,v in d['rooflines'].items()})"; }
for i in 1 2; do b pf0; SPL_GEMM_PREFETCH=1 b pf1; done
SPL_GEMM_PREFETCH=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tc -c 12 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null > gpurun_out/pf1.csv
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tc -c 12 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null > gpurun_out/pf0.csv
