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


def _compare_sets(go, gr, ro, rr):
    """Vectorised CorrespondenceSet comparison: per query, identical root sets (same bones in the same
    order); over the identical sets, |Δx| per root, equal iteration counts, and the roots beyond 1e-4
    as (query, bone, GPU x)."""
    cg, cr = np.diff(go), np.diff(ro)
    eq = cg == cr
    q = np.nonzero(eq & (cg > 0))[0]
    cnt = cg[q]
    within = np.arange(int(cnt.sum())) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    ai = np.repeat(go[:-1][q], cnt) + within
    bi = np.repeat(ro[:-1][q], cnt) + within
    bone_eq = gr[ai, 13].view(np.int32) == rr["bone"][bi]
    qbad = np.zeros(go.shape[0] - 1, bool)
    qbad[np.repeat(q, cnt)[~bone_eq]] = True
    same = eq & ~qbad
    ok = ~qbad[np.repeat(q, cnt)]  # roots of identical sets
    d = np.abs(gr[ai, :3] - rr["x"][bi]).max(1)
    dx = float(d[ok].max()) if ok.any() else 0.0
    it_eq = float((gr[ai[ok], 14].view(np.int32) == rr["iters"][bi[ok]]).mean()) if ok.any() else 1.0
    far = np.nonzero(ok & (d > 1e-4))[0]
    outliers = [(int(np.repeat(q, cnt)[k]), int(rr["bone"][bi[k]]), gr[ai[k], :3].copy()) for k in far]
    return int(same.sum()), dx, it_eq, outliers


def _frames_c4(n_poses, n):
    """bench.py's C4 workload (--poses 16 --points 1000000 --grid 64,64,64, rank 0): pose 0 is
    make_scene(seed 1); poses 1.. are seeded random poses with their own uniform points."""
    sc = S.make_scene((64, 64, 64), n, seed=1)
    skel = S.smpl_like_skeleton()
    frames = [(sc.bones, sc.points)]
    for fi in range(1, n_poses):
        rng = np.random.default_rng(1 * 7919 + fi)
        bones = S.forward_kinematics(skel, rng.uniform(-0.5, 0.5, sc.n_bones))
        lo, hi = S.posed_sampling_box(skel, bones, 0.1)
        frames.append((bones.reshape(sc.n_bones, 12).astype(np.float32),
                       S.uniform_points(lo, hi, n, rng).astype(np.float32)))
    return sc, frames


@pytest.mark.parametrize("workload", ["C4", "C5", "C5-uniform"])
def test_full_bench_workloads_equal_reference_sources(deformer, workload):
    """Every solve of the bench's large workloads against the reference's own code: C4 in full (16 poses ×
    1 M points, 64³ — 384 M solves) and the C5 per-GPU shard in full (8 M ray samples, 128×128×32 — 192 M
    solves, in chunks of 2 M queries; solves are independent). Per query: identical root sets on
    >= 99.99 %. Per root: within 1e-4, except where the reference's build itself is ambiguous — a root
    beyond 1e-4 must then be a float64 re-solve equal to the oracle's (the reference's code in its
    explicit-FMA order) to 1e-9: on 40-50-iteration trajectories the oracle and this build of the
    reference's sources (GCC's own contraction, oracle/_ref) part ways."""
    if workload == "C4":
        sc, frames = _frames_c4(16, 1_000_000)
        chunks = [(b, p) for b, p in frames]
    else:  # bench.py's C5: 64 samples per ray; C5-uniform: the same grid with uniform points (round-1 C5)
        sc = S.make_scene((128, 128, 32), 8_000_000, seed=1, points="rays" if workload == "C5" else "uniform")
        chunks = [(sc.bones, sc.points[c:c + 2_000_000]) for c in range(0, 8_000_000, 2_000_000)]
    o = sc.search_options(50)
    so = SearchOptions(50, o["conv_eps"], o["div_eps"], o["dedup_dist"])
    w = torch.from_numpy(sc.weights).cuda()
    total_q = same_q = 0
    dx_max, it_eqs, far = 0.0, [], []
    for bones, pts in chunks:
        B, x = torch.from_numpy(np.ascontiguousarray(bones)).cuda(), torch.from_numpy(np.ascontiguousarray(pts)).cuda()
        offs, roots = deformer.deform(w, sc.dims, sc.bbox, B, x, so)
        go = offs.cpu().numpy()
        gr = roots[: int(go[-1])].cpu().numpy()
        del offs, roots
        rr = oracle.ref_batch_search(sc.weights, sc.dims, sc.bbox, bones, pts, workers=os.cpu_count() or 8, **o)
        same, dx, it_eq, outl = _compare_sets(go, gr, rr["offsets"], rr)
        total_q += pts.shape[0]
        same_q += same
        dx_max = max(dx_max, dx)
        it_eqs.append(it_eq)
        for q, b, gx in outl:  # the oracle on just that query: the GPU root must be its float64 re-solve
            r1 = oracle.batch_search(sc.weights, sc.dims, sc.bbox, bones, pts[q:q + 1], workers=1, **o)
            far.append((q, b, float(np.abs(gx - r1["x_c"][0, b]).max()), int(r1["iters"][0, b])))
    print(f"\n{workload} in full ({total_q} queries, {total_q * sc.n_bones} solves) vs the reference's own code: "
          f"identical root sets {same_q / total_q:.7f} ({total_q - same_q} queries differ), max|dx| {dx_max:.2e}, "
          f"equal iteration counts {min(it_eqs):.6f}; roots beyond 1e-4: {len(far)} "
          f"(|GPU - oracle| {[f'{d:.1e}' for _, _, d, _ in far]}, oracle iterations {[i for *_, i in far]})")
    assert same_q / total_q >= 0.9999
    assert len(far) <= 1e-6 * total_q * sc.n_bones
    for q, b, d, it in far:
        assert d <= 1e-6 and it >= 20, (q, b, d, it)
