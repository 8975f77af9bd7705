# GPU test suite with the FMA-pipe exponential offload on (default) + forward kernel A/B under ncu
set +e
mkdir -p gpurun_out/poly
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/poly/gputest.log 2>&1; echo pytest $?; tail -3 gpurun_out/poly/gputest.log
for pe in 0 4 0 4; do SPL_ATTN_POLY=$pe timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fa_fwd_pp -c 3 --csv python tools/ab_attn.py 2>/dev/null | grep fa_fwd_pp | awk -F'","' -v pe=$pe '{print "ncu pe=" pe, $NF}'; done
