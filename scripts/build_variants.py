"""Build tuning variants of libfsk_b200.so into build/variants/<name>.so (cross-compiled
here; the .so files travel to the GPU box with the gpurun snapshot). Usage:
    python scripts/build_variants.py name="-DFOO=1 -DBAR=2" name2="..."
then on the box: FSK_LIB=build/variants/<name>.so python bench.py ..."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2211_15601_b200 import build as B  # noqa: E402


def one(name, defs):
    srcs, _ = B._sources()
    out = os.path.join(ROOT, "build", "variants", name + ".so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = ["nvcc", *B.NVCC_FLAGS, *defs.split(), "-shared", "-o", out, *srcs, *B.LIBS]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return name, r.returncode, r.stderr[-2000:]


if __name__ == "__main__":
    jobs = [a.split("=", 1) for a in sys.argv[1:]]
    with ThreadPoolExecutor(4) as ex:
        for name, rc, err in ex.map(lambda j: one(*j), jobs):
            print(name, "ok" if rc == 0 else "FAILED\n" + err)
