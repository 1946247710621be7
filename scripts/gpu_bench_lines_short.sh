# Round-end bench lines only (C2 default with e2e + CPU leg, C3 / C5 / C4), GPU tests, smoke
O=gpurun_out/final4; mkdir -p $O
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 200 $O/bench_c2.json
for c in C3 C5 C4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --cpu-seconds 10 > $O/bench_$c.json 2> $O/bench_$c.err
  tail -c 200 $O/bench_$c.json
done
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
