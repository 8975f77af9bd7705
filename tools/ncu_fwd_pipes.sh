# ncu --set full of the ping-pong attention forward (22B t=1 selective): SASS stall lines plus
# the pipe-utilisation / instruction-mix details (dev tool)
set +e
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fa_fwd_pp" -c 1 \
  -o gpurun_out/fwd_full python tools/ab_attn.py > gpurun_out/ncu_fwd.log 2>&1
echo ncu $?
ncu -i gpurun_out/fwd_full.ncu-rep --page source --csv --print-source sass > gpurun_out/fwd_src.csv 2>/dev/null
python tools/ncu_src_stalls.py gpurun_out/fwd_src.csv 60 > gpurun_out/fwd_stalls.txt 2>&1
ncu -i gpurun_out/fwd_full.ncu-rep --page details --csv > gpurun_out/fwd_details.csv 2>/dev/null
ncu -i gpurun_out/fwd_full.ncu-rep --page raw --csv > gpurun_out/fwd_raw.csv 2>/dev/null
rm -f gpurun_out/fwd_full.ncu-rep
head -30 gpurun_out/fwd_stalls.txt
