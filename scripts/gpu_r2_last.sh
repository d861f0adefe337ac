mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/last_tests.log 2>&1; echo "rc $?" >> gpurun_out/last_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/last_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/last_c2.json 2> gpurun_out/last_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/last_ref.json 2> gpurun_out/last_ref.err
