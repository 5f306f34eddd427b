python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref13.json 2>gpurun_out/ref13.err; tail -2 gpurun_out/ref13.err; cat gpurun_out/ref13.json
/usr/bin/time -v timeout 900 python bench.py > gpurun_out/bench13.json 2>gpurun_out/bench13.err; grep -E "Elapsed|Maximum resident" gpurun_out/bench13.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r5.csv python tools/profile_step.py --steps 1 > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_attn -c 1 -o gpurun_out/attn_r5 python tools/profile_step.py --steps 1 > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_gemm_tc -c 5 -o gpurun_out/gemm_r5 python tools/profile_step.py --steps 1 > /dev/null 2>&1
ls gpurun_out
