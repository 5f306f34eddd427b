timeout 300 python tools/repro.py --reqs 64 --prompt 1300 --layers 2 --steps 8 --rows 8192 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_engine.py -q -p no:cacheprovider 2>&1 | tail -4
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench9.json 2> gpurun_out/bench9.err; tail -3 gpurun_out/bench9.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r4.csv python tools/profile_step.py --steps 1 > gpurun_out/ncu_list4.log 2>&1; tail -1 gpurun_out/ncu_list4.log
