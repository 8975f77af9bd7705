set +e
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q -p no:cacheprovider 2>&1 | tail -1
b() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('$1', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:(round(v['ms_per_step'],2) if v else None) for k,v in d['rooflines'].items()})"; }
b new; b new
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_tc" --csv python tools/t8_gemm_profile.py 2>/dev/null | grep gemm > gpurun_out/t8_gemm_new.csv
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gemm_tc" -c 24 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null > gpurun_out/t1_gemm_new.csv
