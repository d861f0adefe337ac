mkdir -p gpurun_out
python scripts/mlp_bench.py 5 > gpurun_out/mn_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mlp_fwd" -c 3 -o gpurun_out/r02_mlp -f python scripts/mlp_bench.py 2 > gpurun_out/mn_ncu.log 2>&1
