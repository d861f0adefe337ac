mkdir -p gpurun_out
python scripts/sanitize_c1.py > gpurun_out/san_plain.log 2>&1; echo "rc $?" >> gpurun_out/san_plain.log
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python scripts/sanitize_c1.py > gpurun_out/san_memcheck.log 2>&1; echo "rc $?" >> gpurun_out/san_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 50 python scripts/sanitize_c1.py > gpurun_out/san_racecheck.log 2>&1; echo "rc $?" >> gpurun_out/san_racecheck.log
timeout 1500 compute-sanitizer --tool synccheck --print-limit 50 python scripts/sanitize_c1.py > gpurun_out/san_synccheck.log 2>&1; echo "rc $?" >> gpurun_out/san_synccheck.log
