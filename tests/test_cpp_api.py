"""The reference-facing C++ API (include/fskin/*.hpp) compiled into a client program the way
a reference caller would use it, run on the GPU, its CorrespondenceSets compared with the
oracle's kept roots."""
import os
import subprocess

import numpy as np
import pytest

import oracle
from paper_2211_15601_b200 import build as B
from paper_2211_15601_b200 import synthetic as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "fskin_api_check.cpp")


def compile_client(tmp_path):
    B.build()
    exe = str(tmp_path / "fskin_api_check")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
                    B.LIB, f"-Wl,-rpath,{os.path.dirname(B.LIB)}"], check=True)
    return exe


def test_cpp_client_compiles_against_the_api(tmp_path):
    assert os.path.exists(compile_client(tmp_path))


@pytest.mark.gpu
def test_cpp_api_batch_search_matches_oracle(tmp_path):
    exe = compile_client(tmp_path)
    sc = S.make_scene((32, 32, 32), 3000, seed=21, points="training")
    max_iters = 50
    inp = tmp_path / "in.bin"
    with open(inp, "wb") as f:
        np.array([*sc.dims, sc.n_bones, sc.points.shape[0]], np.int32).tofile(f)
        sc.bbox.astype(np.float32).tofile(f)
        np.array([max_iters], np.int32).tofile(f)
        sc.weights.tofile(f)
        sc.bones.tofile(f)
        sc.points.tofile(f)
    out = tmp_path / "sets.txt"
    r = subprocess.run([exe, str(inp), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    ref = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=8,
                              **sc.search_options(max_iters))
    lines = out.read_text().splitlines()
    assert len(lines) == sc.points.shape[0]
    agree, total, maxdx = 0, 0, 0.0
    for p, ln in enumerate(lines):
        f = ln.split()
        k = int(f[0])
        bones = [int(f[1 + 6 * j]) for j in range(k)]
        ref_b = list(np.where(ref["keep"][p] == 1)[0])
        total += 1
        agree += bones == ref_b
        for j, b in enumerate(bones):
            if ref["keep"][p, b]:
                x = np.array([float(v) for v in f[2 + 6 * j:5 + 6 * j]])
                maxdx = max(maxdx, np.abs(x - ref["x_c"][p, b]).max())
    print(f"\nC++ API: identical root sets for {agree}/{total} queries, max|dx| {maxdx:.2e}")
    assert agree / total >= 0.999
    assert maxdx <= 1e-4
