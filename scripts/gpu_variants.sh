set -x
python -m pytest tests -m gpu -q -rf -s -k "backward or golden" > gpurun_out/pytest16.log 2>&1
B="python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e"
$B --backward --deterministic > gpurun_out/bench16_c3det.log 2>&1
