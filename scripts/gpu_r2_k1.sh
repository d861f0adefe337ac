mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_parity.py tests/test_cpp_api.py -q -x -s > gpurun_out/k1_tests.log 2>&1; echo "rc $?" >> gpurun_out/k1_tests.log
for v in base k1v1; do
  if [ $v = base ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 200 > gpurun_out/k1_c2_$v.json 2> gpurun_out/k1_c2_$v.err
  env $L timeout 600 python bench.py --points 8000000 --grid 128,128,32 --steps 10 --warmup 3 --no-cpu-baseline --no-mlp --no-e2e > gpurun_out/k1_c5_$v.json 2> gpurun_out/k1_c5_$v.err
done
timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import bench, argparse
from paper_2211_15601_b200 import synthetic as S
a=argparse.Namespace(max_iters=50); sc=S.make_scene((32,32,32),200000,seed=1)
print(bench.cpp_api_e2e(sc, a))" > gpurun_out/k1_cpp.log 2>&1
