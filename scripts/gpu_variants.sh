# Tuning sweep over build/variants/*.so (scripts/build_variants.py): bitwise-identity hash
# of the C2 forward outputs and a short bench per variant.
mkdir -p gpurun_out
for v in ${VARIANTS:-build/variants/*.so}; do
  n=$(basename $v .so)
  FSK_LIB=$v timeout 300 python scripts/variant_hash.py >> gpurun_out/var_hash.log 2>&1
  FSK_LIB=$v timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/var_$n.log 2>&1
done
