timeout 300 python tools/attn_bench.py 2>&1
for c in 1 2 4 8 16; do echo "RT_ATTN_CHUNKS=$c"; RT_ATTN_CHUNKS=$c timeout 300 python tools/attn_bench.py small 2>&1; done
