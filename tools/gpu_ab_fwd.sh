set +e
for v in 0 1 128; do echo "== SPL_ATTN_FWD_PP=$v"; SPL_ATTN_FWD_PP=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fa_fwd" -c 3 --csv python tools/ab_attn.py 2>/dev/null | grep fa_fwd | awk -F'","' '{print $5, $NF}' | cut -c1-120; done
