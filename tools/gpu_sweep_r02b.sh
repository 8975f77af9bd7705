# Configs sweep, Table-4 layer times and the tiny-config lines at HEAD (one B200)
set +e
O=gpurun_out/r02s
mkdir -p $O
timeout 1200 python tools/sweep.py > $O/sweep.jsonl 2> $O/sweep.err; echo sweep $?
timeout 300 python tools/layer_times.py --t 8 > $O/layer_times_22B_t8.json 2> $O/lt8.err; echo lt8 $?
timeout 300 python bench.py --config tiny --recompute selective > $O/bench_tiny_selective.json 2> $O/tiny.err; echo tiny $?
timeout 300 python bench.py --config tiny --recompute none > $O/bench_tiny_none.json 2>> $O/tiny.err; echo tiny $?
