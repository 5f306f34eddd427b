timeout 600 python -m pytest tests/test_gpu_ops.py -q -k attention -p no:cacheprovider 2>&1 | tail -2
for c in 0 1 2 3 4 6; do echo "RT_ATTN_CHUNKS=$c"; RT_ATTN_CHUNKS=$c timeout 300 python tools/attn_bench.py 2>&1 | head -4; done
