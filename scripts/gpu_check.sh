set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_a.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_a.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_a.log
timeout 600 python bench.py > gpurun_out/bench_a.log 2>&1; echo "bench rc $?" >> gpurun_out/bench_a.log
