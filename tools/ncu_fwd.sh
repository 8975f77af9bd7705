# ncu --set full (with source) of the attention forward of a 22B t=1 selective step
set +e
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fa_fwd" -c 1 \
  -o gpurun_out/fwd_full python tools/ab_attn.py > gpurun_out/ncu_fwd.log 2>&1
echo ncu $?
ncu -i gpurun_out/fwd_full.ncu-rep --page source --csv --print-source sass > gpurun_out/fwd_src.csv 2>/dev/null
python tools/ncu_src_stalls.py gpurun_out/fwd_src.csv > gpurun_out/fwd_stalls.txt 2>&1
head -60 gpurun_out/fwd_stalls.txt
