"""GPU parity against the REFERENCE'S OWN hot-path sources (oracle/_ref: proj/src/{geometry,skinning,
deformer,correspondence}.cpp compiled unmodified against the restated Eigen subset oracle/eigen_shim; see
tests/test_oracle_ref.py): the GPU's CorrespondenceSets — the output of the reference's batch_search — at
the north-star bar: per-query root sets identical on >= 99.99 % of queries (each covers 24 (point, init)
keep decisions), kept roots within 1e-4 abs."""
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2211_15601_b200 import synthetic as S
from paper_2211_15601_b200.deformer import SearchOptions

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (needs /root/reference)")]


def _compare(deformer, sc, max_iters):
    o = sc.search_options(max_iters)
    w, B, x = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (sc.weights, sc.bones, sc.points))
    offs, roots = deformer.deform(w, sc.dims, sc.bbox, B, x, SearchOptions(max_iters, o["conv_eps"], o["div_eps"],
                                                                           o["dedup_dist"]))
    n = sc.points.shape[0]
    go = offs.cpu().numpy()
    gr = roots[: int(go[-1])].cpu().numpy()
    rr = oracle.ref_batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=os.cpu_count() or 8, **o)
    gbone, rbone = gr[:, 13].view(np.int32), rr["bone"]
    same = np.zeros(n, bool)
    dx, it_eq, both = 0.0, 0, 0
    for p in range(n):
        a0, a1, b0, b1 = go[p], go[p + 1], rr["offsets"][p], rr["offsets"][p + 1]
        if a1 - a0 == b1 - b0 and np.array_equal(gbone[a0:a1], rbone[b0:b1]):
            same[p] = True
            if a1 > a0:
                dx = max(dx, float(np.abs(gr[a0:a1, :3] - rr["x"][b0:b1]).max()))
                it_eq += int((gr[a0:a1, 14].view(np.int32) == rr["iters"][b0:b1]).sum())
                both += a1 - a0
    return same.mean(), dx, it_eq / max(both, 1), int((~same).sum())


@pytest.mark.parametrize("dims,n,seed,points,max_iters", [
    ((32, 32, 32), 10_000, 1, "uniform", 10),       # C1, the oracle configuration
    ((32, 32, 32), 200_000, 1, "uniform", 50),      # C2 in full (4.8M solves)
    ((32, 32, 32), 100_000, 4, "training", 50),     # C3's training-shaped points
    ((64, 64, 64), 50_000, 61, "training", 50),     # C4 grid
    ((128, 128, 32), 50_000, 61, "uniform", 50)])   # C5 grid
def test_gpu_correspondence_sets_equal_reference_sources(deformer, dims, n, seed, points, max_iters):
    sc = S.make_scene(dims, n, seed=seed, points=points)
    same, dx, it_eq, diff = _compare(deformer, sc, max_iters)
    print(f"\n{dims} {points} x {n} (max_iters {max_iters}) vs the reference's own code: identical root sets "
          f"{same:.6f} ({diff} queries differ), max|dx| {dx:.2e}, equal iteration counts {it_eq:.6f}")
    assert same >= 0.9999
    assert dx <= 1e-4
