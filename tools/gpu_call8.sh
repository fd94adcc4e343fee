set -x
python tools/sanitize_small.py > gpurun_out/c8_plain.log 2>&1 && tail -2 gpurun_out/c8_plain.log &&
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/r2_sanitizer_memcheck.log 2>&1
echo "memcheck rc=$?"; tail -12 gpurun_out/r2_sanitizer_memcheck.log
