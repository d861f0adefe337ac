# ncu --set full of one launch of the kernel named by $K (regex on the demangled name), C2 bench workload
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$K" -c 1 -o gpurun_out/ncu_$N -f python bench.py --steps 1 --warmup 1 --no-mlp --no-e2e --no-cpu-baseline --no-graph > gpurun_out/ncu_$N.log 2>&1; echo "rc $?" >> gpurun_out/ncu_$N.log
