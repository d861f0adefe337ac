set -x
B="python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/bench15_c2.log 2>&1
$B --backward --deterministic > gpurun_out/bench15_c3det.log 2>&1
$B --backward > gpurun_out/bench15_c3.log 2>&1
