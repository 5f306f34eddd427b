#!/bin/bash
# Regenerate the round's profile evidence on a B200 box (run from the repo root under
# gpurun); outputs land in gpurun_out/final/, then copied into profiles/ by hand.
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/launch_list.csv python tools/profile_step.py --steps 1 > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name regex:k_attn \
  --launch-count 1 -f -o $O/attn python tools/profile_step.py --steps 1 > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name regex:k_gemm \
  --launch-count 5 -f -o $O/gemm python tools/profile_step.py --steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:k_gemm -c 40 -f \
  -o $O/gemm_prefill512 python tools/gemm_once.py 512 > /dev/null 2>&1
timeout 600 python tools/trace_step.py --steps 3 --json $O/trace.json > $O/trace.txt 2>&1
timeout 600 python tools/e2e_profile.py > $O/e2e_rounds.txt 2>&1
timeout 600 python tools/e2e_profile.py trace > $O/e2e_trace.txt 2>&1
timeout 600 python tools/attn_bench.py grid > $O/attn_grid.txt 2>&1
timeout 600 python tools/prefill_tail_bench.py 1,2,3,4,8 > $O/prefill_tail.txt 2>&1
ls -la $O
