set -x
python -m pytest tests -m gpu -q -rf > gpurun_out/pytest11.log 2>&1
python bench.py > gpurun_out/bench11_full.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke11.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench11_ref.log 2>&1
