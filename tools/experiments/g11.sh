TOOL=${TOOL:-memcheck}
timeout 300 python tools/sanitize_cases.py > gpurun_out/san_plain_$TOOL.log 2>&1 && \
timeout 1200 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitizer_$TOOL.log 2>&1
echo "exit $?" >> gpurun_out/sanitizer_$TOOL.log
tail -20 gpurun_out/sanitizer_$TOOL.log
