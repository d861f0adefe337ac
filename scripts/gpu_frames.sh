# frames entry point + exact modes: tests, bench (default and mixed-exact), ncu of both escalation kernels
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_frames.py tests/test_gpu_exact.py -q -rf > gpurun_out/frames_tests.log 2>&1; echo "rc $?" >> gpurun_out/frames_tests.log
timeout 600 python bench.py > gpurun_out/bench_frames.json 2> gpurun_out/bench_frames.err; echo "rc $?" >> gpurun_out/bench_frames.err
timeout 600 python bench.py --precision mixed-exact --no-mlp --no-cpu-baseline > gpurun_out/bench_mixed_exact.json 2> gpurun_out/bench_mixed_exact.err
for v in true false; do
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:escalated<$v>" -c 1 -o gpurun_out/esc_$v -f python scripts/precision_modes.py --steps 1 > gpurun_out/ncu_esc_$v.log 2>&1; echo "rc $?" >> gpurun_out/ncu_esc_$v.log
done
