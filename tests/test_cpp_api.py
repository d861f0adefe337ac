"""The reference-facing C++ API (include/fskin/*.hpp) compiled into a client program the way
a reference caller would use it, run on the GPU, its CorrespondenceSets compared with the
oracle's kept roots at the north-star bar (per (point, init) keep agreement >= 99.99 %,
positions within 1e-4 abs), at the oracle configuration (max_iters 10) and the reference
default (50). The drop-in passes SearchContext::grid's weights to the search, so its float64
re-solves replay the reference's operation order like fsk_deform's."""
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


def _write_input(path, sc, max_iters):
    with open(path, "wb") as f:
        np.array([*sc.dims, sc.n_bones, sc.points.shape[0]], np.int32).tofile(f)
        sc.bbox.astype(np.float32).tofile(f)
        np.array([max_iters], np.int32).tofile(f)
        sc.weights.tofile(f)
        sc.bones.tofile(f)
        sc.points.tofile(f)


def _read_sets(path, n):
    lines = path.read_text().splitlines()
    assert len(lines) == n
    sets = []
    for ln in lines:
        f = ln.split()
        k = int(f[0])
        sets.append([(int(f[1 + 6 * j]), np.array([float(v) for v in f[2 + 6 * j:5 + 6 * j]]), int(f[6 + 6 * j]))
                     for j in range(k)])
    return sets


@pytest.mark.gpu
@pytest.mark.parametrize("max_iters,seed,points", [(10, 21, "uniform"), (50, 22, "training")])
def test_cpp_api_batch_search_matches_oracle(tmp_path, max_iters, seed, points):
    exe = compile_client(tmp_path)
    n = 20_000
    sc = S.make_scene((32, 32, 32), n, seed=seed, points=points)
    inp, out, ist = tmp_path / "in.bin", tmp_path / "sets.txt", tmp_path / "init.bin"
    _write_input(inp, sc, max_iters)
    th_path, ms_path = tmp_path / "mlp_theta.bin", tmp_path / "mlp_sets.txt"
    r = subprocess.run([exe, str(inp), str(out), str(ist), str(th_path), str(ms_path)], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    ref = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=os.cpu_count() or 8,
                              **sc.search_options(max_iters))
    sets = _read_sets(out, n)
    keep = np.zeros_like(ref["keep"])
    same_set, maxdx, iters_eq, both_n = 0, 0.0, 0, 0
    for p, s in enumerate(sets):
        bones = [b for b, _, _ in s]
        keep[p, bones] = 1
        same_set += bones == list(np.where(ref["keep"][p] == 1)[0])
        for b, x, it in s:
            if ref["keep"][p, b]:
                maxdx = max(maxdx, float(np.abs(x - ref["x_c"][p, b]).max()))
                iters_eq += it == ref["iters"][p, b]
                both_n += 1
    per_solve = (keep == ref["keep"]).mean()
    print(f"\nC++ API max_iters {max_iters}: keep agreement per (point, init) {per_solve:.7f}, identical root "
          f"sets {same_set}/{n}, max|dx| {maxdx:.2e}, equal iteration counts {iters_eq}/{both_n}")
    assert per_solve >= 0.9999
    assert same_set / n >= 0.9999
    assert maxdx <= 1e-4
    if oracle.ref_available():  # and against the reference's own sources (oracle/_ref, tests/test_oracle_ref.py)
        rr = oracle.ref_batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=os.cpu_count() or 8,
                                     **sc.search_options(max_iters))
        same_ref = sum([b_ for b_, _, _ in s_] == list(rr["bone"][rr["offsets"][p]:rr["offsets"][p + 1]])
                       for p, s_ in enumerate(sets))
        print(f"C++ API vs the reference's own code: identical root sets {same_ref}/{n}")
        assert same_ref / n >= 0.9999
    # init_states (correspondence.cpp:58-70) through the drop-in: float64, the reference's operation
    # order (weight-grid Jacobian) -> the oracle's values bit for bit
    a = np.fromfile(ist, np.float64)
    nb = sc.n_bones
    rx0, rj0 = oracle.init_states(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points[1:2])
    np.testing.assert_array_equal(a[:3 * nb].reshape(nb, 3), rx0[0])
    np.testing.assert_array_equal(a[3 * nb:].reshape(nb, 3, 3), rj0[0])
    # SearchVariant::Mlp through the API: the reference's SkinningMlp(n_b, seed, domain) init, its search on the
    # tensor cores, vs the oracle's MLP-variant search on the same (float32-rounded) parameters
    theta = np.fromfile(th_path, np.float64).astype(np.float32).astype(np.float64)
    widths = [3, 64, 64, 64, sc.n_bones]
    m = 2000
    mr = oracle.batch_search_mlp(theta, widths, sc.bones, sc.points[:m], workers=os.cpu_count() or 8,
                                 **sc.search_options(max_iters))
    msets = _read_sets(ms_path, m)
    same = sum([b for b, _, _ in s_] == list(np.where(mr["keep"][p] == 1)[0]) for p, s_ in enumerate(msets))
    mdx = max((float(np.abs(x - mr["x_c"][p, b]).max()) for p, s_ in enumerate(msets) for b, x, _ in s_
               if mr["keep"][p, b]), default=0.0)
    print(f"C++ API MLP variant: identical root sets {same}/{m} vs the oracle, max|dx| {mdx:.2e}")
    assert same / m >= 0.999 and mdx <= 1e-4
