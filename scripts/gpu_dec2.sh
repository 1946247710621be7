# fused decoder check: fused vs unfused vs oracle, the decoder / batched GPU tests, a C5
# bench summary and the fused-kernel trace.  Tag in $1.
tag=${1:-d}
timeout 600 python scripts/dec_check.py > gpurun_out/${tag}_check.txt 2>&1; tail -12 gpurun_out/${tag}_check.txt
timeout 900 python -m pytest tests/test_gpu_batched.py -x -q 2>&1 | tail -5
python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c5.json 2> gpurun_out/${tag}_c5.err
python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/{tag}_c5.json").read().strip().splitlines()[-1])
    print("c5", d["value"], d["p50_ms"], "parity", d["parity"] and d["parity"].get("pass"),
          {k: v["ms_per_step"] for k, v in d["stages"].items()})
except Exception as e:
    print("c5 FAILED", e, open(f"gpurun_out/{tag}_c5.err").read()[-1500:])
PY
timeout 300 python scripts/dec_trace.py --config C5 > gpurun_out/${tag}_trace.txt 2>&1; head -40 gpurun_out/${tag}_trace.txt
