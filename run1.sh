set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch; print(torch.cuda.get_device_name(0))"
timeout 300 python -m pytest tests/test_gpu_ops.py -q -x -k "init_weights or priority" -p no:cacheprovider 2>&1 | tail -20
timeout 300 python -m pytest tests/test_gpu_ops.py -q -k "gemm or argmax" -p no:cacheprovider 2>&1 | tail -30
timeout 300 python -m pytest tests/test_gpu_ops.py -q -k "attention" -p no:cacheprovider 2>&1 | tail -30
timeout 600 python -m pytest tests/test_gpu_engine.py -q -k "sched or submit" -p no:cacheprovider 2>&1 | tail -30
timeout 600 python -m pytest tests/test_gpu_engine.py -q -k "tiny" -p no:cacheprovider 2>&1 | tail -30
