#!/usr/bin/env python
"""Regenerate the golden fixtures of tests/golden/.

The reference ships no golden vectors and cannot be run here, so the
fixtures are (1) the SPEC.md known-answer examples written out as vectors and (2) a small
seeded scene with the CPU oracle's outputs, which pins the oracle itself against drift
and gives the GPU tests a fixed target. Run from the repo root:

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2211_15601_b200 import synthetic as S  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def scene_fixture():
    sc = S.make_scene((8, 8, 8), 128, seed=2024, points="training")
    opts = sc.search_options(50)
    r = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=1, **opts)
    np.savez_compressed(
        os.path.join(OUT, "scene_small.npz"),
        dims=np.array(sc.dims, np.int32), bbox=sc.bbox, weights=sc.weights, bones=sc.bones, points=sc.points,
        max_iters=np.int32(50), conv_eps=opts["conv_eps"], div_eps=opts["div_eps"], dedup_dist=opts["dedup_dist"],
        x_c=r["x_c"], iters=r["iters"].astype(np.uint8), converged=r["converged"], keep=r["keep"])


def kat_fixture():
    """SPEC.md examples as explicit input/expected pairs."""
    t1 = np.eye(3, 4)
    t1[:, 3] = [1, 0, 0]
    t2 = np.eye(3, 4)
    t2[:, 3] = [0, 1, 0]
    kats = {
        # weights (0.5, 0.5), B1 = translation (1,0,0), B2 = translation (0,1,0)
        "lbs_blend_translation": {"weights": [0.5, 0.5], "bones": [t1.ravel().tolist(), t2.ravel().tolist()],
                                  "expected": (0.5 * t1 + 0.5 * t2).ravel().tolist()},
        # n_b = 2, B1 = translation (1,0,0), B2 = identity, x' = (1.5,0,0)
        "init_states_two_bone": {"bones": [t1.ravel().tolist(), np.eye(3, 4).ravel().tolist()],
                                 "x_prime": [1.5, 0.0, 0.0], "expected_x0": [[0.5, 0, 0], [1.5, 0, 0]]},
        # dedup
        "dedup_identical": {"roots": [[0, 0, 0], [0, 0, 0]], "dist": 0.1, "expected_keep": [1, 0]},
        "dedup_two_apart": {"roots": [[0, 0, 0], [0.2, 0, 0]], "dist": 0.1, "expected_keep": [1, 1]},
        # correspondence.cpp:168 strict '<': a root exactly dedup_dist away survives
        "dedup_strict_boundary": {"roots": [[0, 0, 0], [0.5, 0, 0]], "dist": 0.5, "expected_keep": [1, 1]},
    }
    with open(os.path.join(OUT, "kats.json"), "w") as f:
        json.dump(kats, f, indent=1)


if __name__ == "__main__":
    scene_fixture()
    kat_fixture()
    print("wrote", os.listdir(OUT))
