# Sweeps on the final build: token-chain tile rows (DR_TOK_ROWS) at C2 / C5, attention plans at C4
O=gpurun_out/sweep; mkdir -p $O
run() { timeout 300 python bench.py --config $1 --steps $2 --warmup 5 --no-e2e --no-cpu-baseline --no-parity > $O/b.json 2>/dev/null; python -c "import json;d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]);print('$3', '$1', d['value'], d['p50_ms'])"; }
for r in 0 64; do if [ $r = 0 ]; then unset DR_TOK_ROWS; else export DR_TOK_ROWS=$r; fi; run C2 300 "tok_rows=$r"; done
unset DR_TOK_ROWS
for r in 0 64; do if [ $r = 0 ]; then unset DR_TOK_ROWS; else export DR_TOK_ROWS=$r; fi; run C5 15 "tok_rows=$r"; done
unset DR_TOK_ROWS
for v in "0 0" "4 1" "4 2" "4 4" "2 1" "2 2" "2 4" "1 1" "1 2"; do set -- $v; export DR_ATTN_QT=$1 DR_ATTN_KSPLIT=$2; run C4 60 "qt=$1,k=$2"; done
