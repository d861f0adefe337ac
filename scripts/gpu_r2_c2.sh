mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_frames.py tests/test_gpu_mlp.py tests/test_gpu_mlp_variant.py -q -x > gpurun_out/c2b_tests.log 2>&1; echo "rc $?" >> gpurun_out/c2b_tests.log
timeout 900 python bench.py > gpurun_out/c2b.json 2> gpurun_out/c2b.err
