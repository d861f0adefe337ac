for c in 1 2 3 4; do
FSK_HOST_CHUNKS=$c timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-mlp > gpurun_out/e2e_chunks_$c.log 2>&1
done
FSK_HOST_CHUNKS=3 timeout 600 python -m pytest tests/test_gpu_parity.py -q -rf -k "host" > gpurun_out/pytest_host3.log 2>&1
FSK_HOST_CHUNKS=7 timeout 600 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -q -rf -k "host or multi" > gpurun_out/pytest_host7.log 2>&1
