# tuning sweep: tests on the default build, then bench variants (each rebuilds in place on the box)
set -x
python -m pytest tests -m gpu -q -rf > gpurun_out/pytest10.log 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/bench10_graph.log 2>&1
$B --no-graph > gpurun_out/bench10_nograph.log 2>&1
$B --backward > gpurun_out/bench10_c3.log 2>&1
$B --backward --deterministic > gpurun_out/bench10_c3det.log 2>&1
$B --grid 64,64,64 --points 1000000 --poses 16 --steps 3 > gpurun_out/bench10_c4.log 2>&1
FSK_NVCC_DEFS=-DFSK_ESC_MINB=4 python paper_2211_15601_b200/build.py --force > /dev/null 2>&1 && $B > gpurun_out/bench10_esc4.log 2>&1
FSK_NVCC_DEFS=-DFSK_ESC_MINB=2 python paper_2211_15601_b200/build.py --force > /dev/null 2>&1 && $B > gpurun_out/bench10_esc2.log 2>&1
