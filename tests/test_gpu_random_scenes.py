"""Randomised workloads against the oracle (seeded, so reproducible): grid shapes from 2 to 48 vertices
per axis (anisotropic), point counts from 1 to 6 000 (ragged around the warp and CTA sizes), SMPL-like
and 3-40-bone chain skeletons, pose magnitudes up to 1 rad, uniform / training / ray-sample points,
max_iters 1-60. Each scene at the north-star bar, with the mask bar stated as a flip budget so tiny
scenes are not judged on a fraction of one solve: at most max(1, 1e-4 · solves) converged-mask flips,
and every root both sides converged within 1e-4."""
import numpy as np
import pytest
import torch

import oracle
from paper_2211_15601_b200 import synthetic as S
from paper_2211_15601_b200.deformer import SearchOptions

pytestmark = pytest.mark.gpu


def _scene(seed):
    rng = np.random.default_rng(1000 + seed)
    dims = tuple(int(v) for v in rng.integers(2, 49, 3))
    n = int(rng.choice([1, 31, 33, 127, 129, 257, 1000, 3000, 6000]))
    skel = S.smpl_like_skeleton() if rng.random() < 0.5 else S.chain_skeleton(int(rng.integers(3, 41)))
    pose = rng.uniform(-1.0, 1.0, skel.bone_count) * rng.uniform(0.1, 1.0)
    points = str(rng.choice(["uniform", "training", "rays"]))
    max_iters = int(rng.choice([1, 3, 8, 9, 10, 25, 50, 60]))
    sc = S.make_scene(dims, n, seed=seed, pose=pose, points=points, skeleton=skel)
    return sc, max_iters


@pytest.mark.parametrize("seed", range(24))
def test_random_scene_against_oracle(deformer, seed):
    sc, max_iters = _scene(seed)
    o = sc.search_options(max_iters)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    w, B, x = dev(sc.weights), dev(sc.bones), dev(sc.points)
    tg64 = torch.empty((w.shape[0], 12), dtype=torch.float64, device="cuda")
    tg = deformer.precompute_transform_grid(w, sc.dims, sc.bbox, B, out64=tg64)
    out = deformer.batch_search(tg, sc.dims, sc.bbox, B, x, SearchOptions(max_iters, o["conv_eps"], o["div_eps"],
                                                                          o["dedup_dist"]), tgrid64=tg64, weights=w)
    g = {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}
    r = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=8, **o)
    solves = g["converged"].size
    flips = int((g["converged"] != r["converged"]).sum())
    both = (g["converged"] == 1) & (r["converged"] == 1)
    dx = float(np.abs(g["x_c"] - r["x_c"])[both].max()) if both.any() else 0.0
    tol = 1e-4
    print(f"\nseed {seed}: {sc.dims} n={sc.points.shape[0]} bones={sc.n_bones} max_iters={max_iters} "
          f"solves={solves} flips={flips} max|dx|={dx:.2e} (tol {tol:.1e})")
    assert flips <= max(1, int(1e-4 * solves))
    assert dx <= tol
