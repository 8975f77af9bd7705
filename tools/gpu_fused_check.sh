set +e
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_widths.py -x -q -p no:cacheprovider -k 22B > gpurun_out/fc_widths.log 2>&1; echo widths $?
tail -2 gpurun_out/fc_widths.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fc_bench_0.json 2> gpurun_out/fc_bench_0.err; echo bench $?
python - <<'PY'
import json
d=json.loads(open("gpurun_out/fc_bench_0.json").read().strip().splitlines()[-1])
print(round(d["value"]), d["ms_per_step"], d["rooflines"]["attention"]["ms_per_step"], d["rooflines"]["other"]["ms_per_step"])
PY
SPL_ATTN_TRACE=1 timeout 200 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --no-graphs 2>&1 | grep -v "^{" | head -14
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fa_bwd_fused" -c 2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep -E "fa_bwd|gpu__time"
