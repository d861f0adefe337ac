"""bench.py's workload selection (CPU): the C5 grid defaults to BASELINE configs[4]'s dense ray samples,
everything else to uniform points; per-rank shards follow the same distribution; the workload string
names it (the driver compares both arms' `config`)."""
import argparse
import importlib.util
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_under_test", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def _args(**kw):
    a = dict(grid="32,32,32", poses=1, backward=False, points_dist="auto", points=640, max_iters=50, seed=1)
    a.update(kw)
    return argparse.Namespace(**a)


def test_points_distribution_per_workload():
    b = _bench()
    assert b.points_dist(_args()) == "uniform"
    assert b.points_dist(_args(grid="128,128,32")) == "rays"
    assert b.points_dist(_args(grid="128,128,32", poses=2)) == "uniform"
    assert b.points_dist(_args(grid="128,128,32", points_dist="training")) == "training"
    assert "rays, 64 samples per ray" in b.workload_name(_args(grid="128,128,32"))
    assert b.workload_name(_args()).startswith("C2")
    assert b.workload_name(_args(backward=True)).startswith("C3")
    assert b.workload_name(_args(poses=16)).startswith("C4")


def test_rank_shards_are_distinct_and_follow_the_distribution():
    b = _bench()
    a = _args(grid="128,128,32")
    s0, s1 = b.scene_for_rank(a, 0), b.scene_for_rank(a, 1)
    assert s0.points.shape == s1.points.shape == (640, 3)
    assert not np.array_equal(s0.points, s1.points)
    # ray samples: consecutive points of one ray are collinear (64 samples per ray)
    for sc in (s0, s1):
        p = sc.points[:64].astype(np.float64)
        d = p[1:] - p[:-1]
        cos = (d[1:] * d[:-1]).sum(1) / (np.linalg.norm(d[1:], axis=1) * np.linalg.norm(d[:-1], axis=1))
        assert (cos > 0.999).all()
