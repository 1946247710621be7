# Quick check of the current build on one B200: GPU tests, smoke, C2 and C5 bench lines.
O=gpurun_out/verify; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 1500 $O/bench_c2.json
timeout 900 python bench.py --config C5 --steps 20 --warmup 5 --cpu-seconds 5 > $O/bench_C5.json 2> $O/bench_C5.err; tail -c 1500 $O/bench_C5.json
