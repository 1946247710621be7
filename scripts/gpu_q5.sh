tag=${1:-q5}
bash scripts/gpu_dec2.sh $tag
for c in C2 C5; do
DR_B200_LIB=paper_2509_10466_b200/_build_mth32/libdrb200.so python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/${tag}_mth32_$c.json 2>/dev/null
python -c "import json,sys;d=json.loads(open('gpurun_out/${tag}_mth32_$c.json').read().strip().splitlines()[-1]);print('mth32 $c', d['value'], d['stages']['mask_stage'])"
done
