time (timeout 900 python bench.py > gpurun_out/bench14.json 2>gpurun_out/bench14.err)
python tools/profile_step.py --steps 1 2>&1 | tail -1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r6.csv python tools/profile_step.py --steps 1 > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_gemm_tc -c 5 -o gpurun_out/gemm_r6 python tools/profile_step.py --steps 1 > /dev/null 2>&1
