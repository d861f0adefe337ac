# GPU suite + default bench (round 2)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf -s > gpurun_out/r2_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-mlp > gpurun_out/r2_c2.json 2> gpurun_out/r2_c2.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "rc $?" >> gpurun_out/r2_smoke.log
