# host-path rgb upload chunking A/B (DR_RGB_CHUNKS), graph on; GPU tests first
set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
for c in 1 2 4; do
DR_RGB_CHUNKS=$c timeout 300 python scripts/e2e_trace.py > gpurun_out/e2e_trace_c$c.txt 2>&1
done
for i in 1 2 3; do for c in 1 2 4; do
DR_RGB_CHUNKS=$c timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c${c}_$i.json 2> gpurun_out/bench_c${c}_$i.err
done; done
cat gpurun_out/pytest_gpu.log
