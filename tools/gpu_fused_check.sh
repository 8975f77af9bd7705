set +e
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_widths.py -x -q -k "22B" -p no:cacheprovider > gpurun_out/fc_widths.log 2>&1; echo widths $?
tail -3 gpurun_out/fc_widths.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fc_bench_fused.json 2> gpurun_out/fc_bench_fused.err; echo bench_fused $?
SPL_ATTN_DETERMINISTIC=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fc_bench_split.json 2> gpurun_out/fc_bench_split.err; echo bench_split $?
python - <<'PY'
import json
for n in ("fused","split"):
    try:
        d=json.loads(open(f"gpurun_out/fc_bench_{n}.json").read().strip().splitlines()[-1])
        print(n, round(d["value"]), d["ms_per_step"], d["rooflines"]["attention"])
    except Exception as e: print(n, "ERR", e)
PY
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fc_gputest.log 2>&1; echo gputest $?
tail -30 gpurun_out/fc_gputest.log
