# default mode = exact-replay escalation: full GPU suite, smoke, bench (default + mixed-fast)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_all.log 2>&1; echo "rc $?" >> gpurun_out/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --precision mixed-fast --no-mlp --no-cpu-baseline > gpurun_out/bench_fast.json 2> gpurun_out/bench_fast.err
