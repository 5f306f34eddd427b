for cfg in "--reqs 64 --prompt 1300 --layers 2 --steps 8 --rows 8192" "--reqs 64 --prompt 1300 --layers 2 --steps 8 --rows 4096" "--reqs 16 --prompt 1300 --layers 1 --steps 4 --rows 8192" "--reqs 64 --prompt 100 --layers 1 --steps 4 --rows 8192"; do
  echo "== $cfg"; timeout 300 python tools/repro.py $cfg 2>&1 | tail -2
done
timeout 1200 compute-sanitizer --tool memcheck --print-limit 3 python tools/repro.py --reqs 16 --prompt 1300 --layers 1 --steps 3 --rows 8192 2>&1 | grep -v "Host Frame" | head -40
