# host-path rgb upload: event join vs device flag (launch before staging), x chunks; GPU tests first
set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
for v in 0_1 1_1 1_2; do
DR_RGB_FLAG=${v%_*} DR_RGB_CHUNKS=${v#*_} timeout 300 python scripts/e2e_trace.py > gpurun_out/e2e_trace_$v.txt 2>&1
done
for i in 1 2 3; do for v in 0_1 1_1 1_2; do
DR_RGB_FLAG=${v%_*} DR_RGB_CHUNKS=${v#*_} timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_${v}_$i.json 2> gpurun_out/bench_${v}_$i.err
done; done
cat gpurun_out/pytest_gpu.log
