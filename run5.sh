timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_engine.py -q -x -p no:cacheprovider 2>&1 | tail -5
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; tail -3 gpurun_out/bench5.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r3.csv python tools/profile_step.py --steps 1 > gpurun_out/ncu_list3.log 2>&1; tail -1 gpurun_out/ncu_list3.log
