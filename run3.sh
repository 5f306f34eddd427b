set -x
timeout 300 python -m pytest tests/test_gpu_engine.py -q -k llama8b -p no:cacheprovider 2>&1 | tail -5
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -3 gpurun_out/bench3.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python tools/profile_step.py --steps 1 > gpurun_out/ncu_list.log 2>&1; tail -2 gpurun_out/ncu_list.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_attn -c 1 -o gpurun_out/attn_r1 python tools/profile_step.py --steps 1 > gpurun_out/ncu_attn.log 2>&1; tail -2 gpurun_out/ncu_attn.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_gemm_tc -c 4 -o gpurun_out/gemm_r1 python tools/profile_step.py --steps 1 > gpurun_out/ncu_gemm.log 2>&1; tail -2 gpurun_out/ncu_gemm.log
ls -la gpurun_out
