timeout 900 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err
