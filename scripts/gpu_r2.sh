#!/bin/bash
# round-2 GPU check: tests, then C2 / C5 / C3 bench lines (tag in $1)
tag=${1:-x}
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/${tag}_pytest.log
python bench.py --steps 50 --warmup 10 --no-e2e --cpu-seconds 2 > gpurun_out/${tag}_c2.json 2> gpurun_out/${tag}_c2.err
python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c5.json 2> gpurun_out/${tag}_c5.err
python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c3.json 2> gpurun_out/${tag}_c3.err
tail -2 gpurun_out/${tag}_pytest.log
for c in c2 c5 c3; do python - "$tag" "$c" <<'PY'
import json, sys
tag, c = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/{tag}_{c}.json").read().strip().splitlines()[-1])
    st = {k: v["ms_per_step"] for k, v in d["stages"].items()}
    print(c, d["value"], d["p50_ms"], "parity", d["parity"] and d["parity"].get("pass"),
          "roof", d["roofline"]["frac"], d["roofline"].get("mufu", {}).get("frac"), st)
except Exception as e:
    print(c, "FAILED", e, open(f"gpurun_out/{tag}_{c}.err").read()[-1500:])
PY
done
