# does k_dedup re-read the search planes from DRAM in a real (warm) run, and does an L2 set-aside change it?
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-mlp --no-graph"
timeout 600 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:"k_dedup|k_search_fast|k_emit" -c 9 --csv $B > gpurun_out/l2_ncu_default.csv 2> gpurun_out/l2_ncu_default.err
for mb in 0 64 100; do
  FSK_LIB=build/variants/l2p.so FSK_L2_PERSIST_MB=$mb timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 200 > gpurun_out/l2_c2_$mb.json 2> gpurun_out/l2_c2_$mb.err
done
FSK_LIB=build/variants/l2p.so FSK_L2_PERSIST_MB=100 timeout 600 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:"k_dedup|k_search_fast|k_emit" -c 9 --csv $B > gpurun_out/l2_ncu_100.csv 2> gpurun_out/l2_ncu_100.err
