mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_frames.py tests/test_gpu_wire.py tests/test_cpp_api.py tests/test_gpu_exact.py -q -x > gpurun_out/graph_tests.log 2>&1; echo "rc $?" >> gpurun_out/graph_tests.log
for v in 0 1 0 1; do
  FSK_PIPE_GRAPH=$v timeout 600 python bench.py --no-cpu-baseline --no-mlp --steps 100 >> gpurun_out/graph_c2_$v.json 2>> gpurun_out/graph_c2_$v.err
done
