timeout 600 python tools/repro.py --layers 1 --reqs 8 --prompt 300 --steps 4 2>&1 | tail -3
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python tools/repro.py --layers 1 --reqs 8 --prompt 300 --steps 3 2>&1 | grep -v "^=========     Host Frame" | head -60
