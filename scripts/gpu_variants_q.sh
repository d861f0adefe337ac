# quick variant timing: bench (no MLP / CPU / e2e) per build/variants/*.so
mkdir -p gpurun_out; rm -f gpurun_out/var_*
for v in ${VARIANTS:-build/variants/*.so}; do
  n=$(basename $v .so)
  FSK_LIB=$v timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-mlp $BENCH_ARGS > gpurun_out/var_$n.json 2>&1
done
