for v in _build_trace _build_trace_noepi _build_trace_nostream _build_trace_both; do
  echo "== $v"; DEC_TRACE_BUILD=$v timeout 300 python scripts/dec_trace.py --config C5 2>&1 | grep -E "main loop|finish pass|MMA wait"
done
timeout 300 python scripts/token_trace.py --config C5 2>&1 | tail -8
