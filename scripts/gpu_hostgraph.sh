# host-path CUDA graph A/B: GPU tests, e2e trace, bench with DR_HOST_GRAPH=0 / 1
set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
DR_HOST_GRAPH=0 timeout 300 python scripts/e2e_trace.py > gpurun_out/e2e_trace_g0.txt 2>&1
timeout 300 python scripts/e2e_trace.py > gpurun_out/e2e_trace_g1.txt 2>&1
for i in 1 2 3; do
DR_HOST_GRAPH=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_g0_$i.json 2> gpurun_out/bench_g0_$i.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_g1_$i.json 2> gpurun_out/bench_g1_$i.err
done
cat gpurun_out/pytest_gpu.log
