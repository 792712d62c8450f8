# compute-sanitizer over the small (C1 / T-config) GPU parity tests: every librtgs kernel runs at least
# once under each tool.  One gpurun call; summaries land in gpurun_out/sanitize_*.log
set -u
TESTS="tests/test_gpu_parity.py tests/test_gpu_backward.py tests/test_gpu_render_span.py tests/test_gpu_state.py tests/test_gpu_insert.py tests/test_gpu_icp.py tests/test_gpu_decode.py tests/test_gpu_cache.py tests/test_gpu_fused_adam.py"
SEL="${SAN_SEL:-C1 or T3 or bitexact or decode or degenerate or state or insert or icp_parity or fused}"
for tool in memcheck racecheck synccheck initcheck; do
  timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool --error-exitcode 0 --print-limit 50 \
      --target-processes all python -m pytest $TESTS -q -x -k "$SEL" -p no:cacheprovider \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$? $(grep -c 'ERROR SUMMARY' gpurun_out/sanitize_$tool.log) summaries; $(grep -E 'ERROR SUMMARY' gpurun_out/sanitize_$tool.log | sort | uniq -c | head -5)"
  grep -E "passed|failed" gpurun_out/sanitize_$tool.log | tail -1
done
