set -x
python -m pytest tests -m gpu -q -rf -s -k "backward or golden" > gpurun_out/pytest14.log 2>&1
B="python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e"
$B --backward > gpurun_out/bench14_c3.log 2>&1
$B --backward --deterministic > gpurun_out/bench14_c3det.log 2>&1
