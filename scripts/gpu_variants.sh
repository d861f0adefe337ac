# tuning sweep: tests on the default build, then bench variants (each rebuilds in place on the box)
set -x
python -m pytest tests -m gpu -q -rf > gpurun_out/pytest9.log 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/bench9_default.log 2>&1
FSK_NVCC_DEFS=-DFSK_ESC_MINB=2 python paper_2211_15601_b200/build.py --force > /dev/null 2>&1 && $B > gpurun_out/bench9_esc2.log 2>&1
