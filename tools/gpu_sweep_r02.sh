set +e
O=gpurun_out/r02
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo pytest $?; tail -2 $O/gputest.log
timeout 900 python tools/sweep.py > $O/sweep.jsonl 2> $O/sweep.err; echo sweep $?
timeout 300 python tools/layer_times.py --t 8 > $O/layer_times_22B_t8.json 2> $O/lt8.err; echo lt8 $?; tail -3 $O/lt8.err
timeout 300 python tools/layer_times.py --t 1 > $O/layer_times_22B_t1.json 2> $O/lt1.err; echo lt1 $?
