set -x
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_engine.py -q -p no:cacheprovider 2>&1 | tail -30
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -5 gpurun_out/bench2.err
cat gpurun_out/bench2.json
