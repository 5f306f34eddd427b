#!/bin/bash
# Regenerate the round's profile evidence on a B200 box (run from the repo root under
# gpurun); outputs land in gpurun_out/final/, then copied into profiles/ by hand.
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/launch_list.csv python tools/profile_step.py --steps 1 > $O/launch_list.out 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name regex:k_attn \
  --launch-count 1 -f -o $O/attn python tools/profile_step.py --steps 1 > $O/attn.out 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name regex:"k_gemm|k_resid" \
  --launch-count 6 -f -o $O/gemm python tools/profile_step.py --steps 1 > $O/gemm.out 2>&1
timeout 600 python tools/trace_step.py --workload C3 --steps 2 > $O/trace_c3.txt 2>&1
timeout 600 python tools/trace_step.py --workload C2 --steps 3 > $O/trace_c2.txt 2>&1
python tools/ncu_summary.py $O/attn.ncu-rep > $O/attn_summary.json 2>&1
# the captured launch's own algorithmic bytes (profile_step prints them) -> bench's traffic ratio
python - $O/attn.out $O/attn_summary.json <<'PY'
import json, re, sys
m = re.search(r"attention algorithmic bytes per layer launch: (\d+)", open(sys.argv[1]).read())
d = json.load(open(sys.argv[2]))
for k in d:
    if m and "k_attn" in k["Kernel Name"]:
        k["alg_bytes_per_launch"] = int(m.group(1))
json.dump(d, open(sys.argv[2], "w"), indent=4)
PY
python tools/ncu_summary.py $O/gemm.ncu-rep > $O/gemm_summary.json 2>&1
ls -la $O
