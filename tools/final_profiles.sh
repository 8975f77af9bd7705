set +e
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 400 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench $?
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref $?
timeout 600 python tools/sweep.py > gpurun_out/sweep_final.jsonl 2> gpurun_out/sweep_final.err; echo sweep $?
timeout 300 python tools/layer_times.py --t 8 > gpurun_out/lt8_final.json 2>/dev/null; echo lt8 $?
timeout 300 python tools/layer_times.py --t 1 > gpurun_out/lt1_final.json 2>/dev/null; echo lt1 $?
timeout 900 python tools/window_bench.py > gpurun_out/window_final.jsonl 2>/dev/null; echo wb $?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_dram_final.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1; echo ncu1 $?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fa_fwd_umma|fa_bwd_dkdv_umma|fa_bwd_dq_umma|keep_bits_k|gemm_tc_pair_kernel|bdr_v|ln_bwd_dx_v" -c 24 -o /tmp/full_final python bench.py --steps 1 --warmup 1 > /dev/null 2>&1; echo ncu2 $?
python tools/ncu_full_summary.py /tmp/full_final.ncu-rep > gpurun_out/ncu_full_final.txt; echo sum $?
