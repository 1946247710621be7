#!/bin/bash
# A/B of the MUFU-offload share (POLY_EVERY) of the attention softmax
for v in _build _build_p2 _build_p4 _build_p0; do
  for cfg in C2 C5; do
    DR_B200_LIB=paper_2509_10466_b200/$v/libdrb200.so python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/poly_${v}_$cfg.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/poly_${v}_$cfg.json').read().strip().splitlines()[-1]); st={k:round(v['ms_per_step'],4) for k,v in d['stages'].items() if 'attn' in k}
print('$v $cfg', d['value'], d['p50_ms'], st)"
  done
done
