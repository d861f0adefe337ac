# quick check: exact + parity tests, bench default and mixed-fast (no MLP, no CPU baseline)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_exact.py tests/test_gpu_parity.py tests/test_gpu_frames.py -q -rf -x > gpurun_out/quick_tests.log 2>&1; echo "rc $?" >> gpurun_out/quick_tests.log
timeout 600 python bench.py --no-mlp --no-cpu-baseline > gpurun_out/bench_q_default.json 2> gpurun_out/bench_q_default.err
timeout 600 python bench.py --precision mixed-fast --no-mlp --no-cpu-baseline > gpurun_out/bench_q_fast.json 2> gpurun_out/bench_q_fast.err
