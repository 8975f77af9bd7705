# Evidence at HEAD after the attention MMA-issue and exponential-offload changes (one B200)
set +e
O=gpurun_out/r02h
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo pytest $?; tail -2 $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo smoke $?
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo bench $?
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo ref $?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_dram.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu1 $?
python tools/profile_summary.py $O/launches_dram.csv $O/ncu_dram_22B_t1_selective.json > $O/ncu_dram_22B_t1_selective.txt 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"fa_fwd_pp|fa_bwd_fused_umma|keep_bits_k|gemm_tc_pair_kernel|bdr_v|ln_bwd_dx_v|ln_fwd_v" -c 20 -o $O/full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu2 $?
python tools/ncu_full_summary.py $O/full.ncu-rep > $O/ncu_full_22B_t1_selective.txt 2>&1
rm -f $O/full.ncu-rep
timeout 300 python tools/layer_times.py --t 1 > $O/layer_times_22B_t1.json 2> $O/lt1.err; echo lt1 $?
