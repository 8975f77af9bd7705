# verification pass on one B200: GPU tests, smoke, bench (own arm + reference arm), launch list
set +e
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo pytest $?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
tail -c 3000 gpurun_out/bench.json
