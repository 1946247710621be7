for v in _build_trace_both _build_trace_both_nomma _build_trace_both_mma2; do
  echo "== $v"; DEC_TRACE_BUILD=$v timeout 300 python scripts/dec_trace.py --config C5 2>&1 | grep -E "main loop|MMA wait|^     [0-3]:"
done
