# full GPU suite, the default bench line (with CPU baseline, e2e, MLP stages) and the reference arm
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf -s > gpurun_out/r2_full_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2_full_tests.log
timeout 900 python bench.py > gpurun_out/r2_full_c2.json 2> gpurun_out/r2_full_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_full_ref.json 2> gpurun_out/r2_full_ref.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_full_smoke.log 2>&1; echo "rc $?" >> gpurun_out/r2_full_smoke.log
lscpu > gpurun_out/r2_lscpu.txt 2>&1; nproc >> gpurun_out/r2_lscpu.txt
