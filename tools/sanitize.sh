mkdir -p gpurun_out/san
for t in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $t --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san/smoke_$t.txt 2>&1
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/repro.py --layers 1 --reqs 140 --prompt 32 --vocab 4096 --steps 4 > gpurun_out/san/repro_$t.txt 2>&1
done
for f in gpurun_out/san/*.txt; do echo "$f: $(tail -2 $f | tr '\n' ' ')"; done
