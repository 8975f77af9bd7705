# ncu --set full (with source) of the fused attention backward of a 22B t=1 selective step
set +e
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fa_bwd_fused" -c 1 \
  -o gpurun_out/bwd_full python tools/ab_attn.py > gpurun_out/ncu_bwd.log 2>&1
echo ncu $?
ncu -i gpurun_out/bwd_full.ncu-rep --page source --csv --print-source sass > gpurun_out/bwd_src.csv 2>/dev/null
python tools/ncu_src_stalls.py gpurun_out/bwd_src.csv > gpurun_out/bwd_stalls.txt 2>&1
head -50 gpurun_out/bwd_stalls.txt
