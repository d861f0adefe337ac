mkdir -p gpurun_out
for k in 1 2 3 4; do
  FSK_HOST_CHUNKS=$k timeout 600 python bench.py --no-cpu-baseline --no-mlp --steps 50 > gpurun_out/ch_c2_$k.json 2> gpurun_out/ch_c2_$k.err
done
