# ncu --set full (with source) of one launch of each attention-side kernel of a 22B t=1 selective step
set +e
mkdir -p gpurun_out
timeout 1500 ncu --set full --import-source on --clock-control none \
  -k regex:"fa_fwd_umma|fa_bwd_fused_umma|keep_bits" -c 4 \
  -o gpurun_out/attn_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_attn.log 2>&1
echo ncu $?
