mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -s -k "full_bench or all_solves or reference_build_spread" > gpurun_out/sg_full.log 2>&1; echo "rc $?" >> gpurun_out/sg_full.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/sg_tests.log 2>&1; echo "rc $?" >> gpurun_out/sg_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-mlp --steps 200 > gpurun_out/sg_c2.json 2> gpurun_out/sg_c2.err
for s in 22 52 82 112; do
  timeout 1500 python scripts/band_study.py $s $((s+30)) > gpurun_out/sg_band_$s.log 2>&1
done
