mkdir -p gpurun_out
timeout 900 python bench.py --poses 16 --points 1000000 --grid 64,64,64 --steps 5 --warmup 3 --no-cpu-baseline --no-mlp > gpurun_out/f3_c4.json 2> gpurun_out/f3_c4.err
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/f3_smoke.log 2>&1
