mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-graph --no-mlp --backward --deterministic"
$B > gpurun_out/dn_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bwd_chunk_reduce|k_bwd_bucket_fill|k_bwd_bucket_count" -c 3 -o gpurun_out/r02_det_bwd -f $B > gpurun_out/dn_ncu.log 2>&1
