"""Synthetic input recipe for the deformer hot path (host side, not timed).

Restates the reference's input generators so the CUDA path and the CPU oracle see
bit-identical float32 inputs:

* 24-bone SMPL-like skeleton with one revolute axis per joint
  (``Bone``/``Skeleton``: ``proj/include/fskin/skeleton.hpp:14-45``),
  ``Skeleton::bone_segment`` (``proj/src/skeleton.cpp:47-62``),
  ``forward_kinematics`` (``proj/src/skeleton.cpp:64-86``) with
  ``RigidTransform::about_axis`` (``proj/src/geometry.cpp:7-14``, Rodrigues).
* ``CapsuleBody::from_skeleton`` / ``canonical_bounds`` / ``posed_bounds``
  (``proj/src/shape.cpp:21-35,104-119``), ``canonical_domain`` and
  ``posed_sampling_box`` (``proj/src/diff.cpp:128-137``).
* ``analytic_weight_grid`` (``proj/tools/fskin_cli.cpp:277-300``): softmax of the
  per-bone max of −d(x, capsule segment)²/τ, τ = (0.1·diag)².
* Uniform posed queries (``fskin_cli.cpp:629-637``) and the training-shaped
  half-uniform / half-near-surface mix (``diff.cpp:148-182``,
  ``shape.cpp:134-175``).

Random streams are numpy's (seeded ``np.random.default_rng``), not libstdc++'s
``mt19937_64`` distributions, so values differ from the reference CLI's draws;
the recipe (boxes, distributions, temperatures) is the same.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# SMPL kinematic tree.
SMPL_PARENTS = [-1, 0, 0, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 9, 9, 12, 13, 14, 16, 17, 18, 19, 20, 21]
SMPL_NAMES = [
    "pelvis", "l_hip", "r_hip", "spine1", "l_knee", "r_knee", "spine2", "l_ankle", "r_ankle",
    "spine3", "l_foot", "r_foot", "neck", "l_collar", "r_collar", "head", "l_shoulder",
    "r_shoulder", "l_elbow", "r_elbow", "l_wrist", "r_wrist", "l_hand", "r_hand",
]
# Approximate T-pose joint positions (metres, y up, ~1.7 m tall).
SMPL_JOINTS = np.array([
    [0.000, 0.930, 0.000], [0.060, 0.840, 0.000], [-0.060, 0.840, 0.000], [0.000, 1.040, -0.010],
    [0.100, 0.470, 0.010], [-0.100, 0.470, 0.010], [0.000, 1.170, 0.000], [0.090, 0.070, -0.030],
    [-0.090, 0.070, -0.030], [0.000, 1.230, 0.020], [0.110, 0.020, 0.100], [-0.110, 0.020, 0.100],
    [0.000, 1.450, -0.010], [0.070, 1.380, 0.000], [-0.070, 1.380, 0.000], [0.000, 1.520, 0.040],
    [0.180, 1.410, -0.010], [-0.180, 1.410, -0.010], [0.440, 1.400, -0.030], [-0.440, 1.400, -0.030],
    [0.700, 1.410, -0.030], [-0.700, 1.410, -0.030], [0.780, 1.400, -0.040], [-0.780, 1.400, -0.040],
])
# One revolute axis per joint: flexion (x) for legs/spine/neck, abduction (z) at
# collars/shoulders, elbow/wrist flexion about y (arms lie along x).
SMPL_AXES = np.array([
    [0, 1, 0], [1, 0, 0], [1, 0, 0], [1, 0, 0], [1, 0, 0], [1, 0, 0], [0, 1, 0], [1, 0, 0],
    [1, 0, 0], [0, 0, 1], [1, 0, 0], [1, 0, 0], [1, 0, 0], [0, 0, 1], [0, 0, 1], [1, 0, 0],
    [0, 0, 1], [0, 0, 1], [0, 1, 0], [0, 1, 0], [0, 1, 0], [0, 1, 0], [0, 0, 1], [0, 0, 1],
], dtype=np.float64)
SMPL_RADII = np.array([
    0.12, 0.09, 0.09, 0.12, 0.06, 0.06, 0.12, 0.045, 0.045, 0.12, 0.04, 0.04,
    0.05, 0.05, 0.05, 0.10, 0.05, 0.05, 0.04, 0.04, 0.04, 0.04, 0.04, 0.04,
])
LEAF_LENGTH = {10: 0.10, 11: 0.10, 15: 0.20, 22: 0.08, 23: 0.08}


@dataclass
class Skeleton:
    """Mirror of ``fskin::Skeleton`` (skeleton.hpp:14-45)."""
    parents: list
    joints: np.ndarray          # [n,3]
    axes: np.ndarray            # [n,3]
    lengths: np.ndarray         # [n]
    radii: np.ndarray           # [n]
    names: list = field(default_factory=list)

    @property
    def bone_count(self) -> int:
        return len(self.parents)

    def validate(self) -> None:  # skeleton.cpp:22-45
        n = self.bone_count
        if n < 1:
            raise ValueError("Skeleton: at least one bone required")
        for i, p in enumerate(self.parents):
            if p >= n or p == i:
                raise ValueError(f"Skeleton: bone {i} has invalid parent")
            if np.linalg.norm(self.axes[i]) < 1e-12:
                raise ValueError(f"Skeleton: bone {i} has degenerate axis")
            if not self.lengths[i] > 0.0:
                raise ValueError(f"Skeleton: bone {i} has non-positive length")
            q, steps = p, 0
            while q >= 0:
                steps += 1
                if q == i or steps > n:
                    raise ValueError("Skeleton: parent indices contain a cycle")
                q = self.parents[q]

    def bone_segment(self, i: int):  # skeleton.cpp:47-62
        j = self.joints[i]
        child = next((c for c in range(self.bone_count) if self.parents[c] == i), -1)
        p = self.parents[i]
        if child >= 0 and np.linalg.norm(self.joints[child] - j) > 1e-9:
            d = self.joints[child] - j
            d = d / np.linalg.norm(d)
        elif p >= 0 and np.linalg.norm(j - self.joints[p]) > 1e-9:
            d = j - self.joints[p]
            d = d / np.linalg.norm(d)
        else:
            a = self.axes[i] / np.linalg.norm(self.axes[i])
            d = np.array([1.0, 0.0, 0.0]) - a[0] * a
            if np.linalg.norm(d) < 1e-6:
                d = np.array([0.0, 1.0, 0.0]) - a[1] * a
            d = d / np.linalg.norm(d)
        return j.copy(), j + self.lengths[i] * d


def smpl_like_skeleton() -> Skeleton:
    n = len(SMPL_PARENTS)
    lengths = np.zeros(n)
    for i in range(n):
        child = next((c for c in range(n) if SMPL_PARENTS[c] == i), -1)
        lengths[i] = (np.linalg.norm(SMPL_JOINTS[child] - SMPL_JOINTS[i]) if child >= 0
                      else LEAF_LENGTH.get(i, 0.08))
    s = Skeleton(list(SMPL_PARENTS), SMPL_JOINTS.copy(), SMPL_AXES.copy(), lengths,
                 SMPL_RADII.copy(), list(SMPL_NAMES))
    s.validate()
    return s


def chain_skeleton(n_bones: int = 3, radius: float = 0.12) -> Skeleton:
    """``builtin_bench_skeleton`` (fskin_cli.cpp:549-562): a chain along +x, axes z."""
    joints = np.array([[float(i), 0.0, 0.0] for i in range(n_bones)])
    axes = np.tile([0.0, 0.0, 1.0], (n_bones, 1))
    return Skeleton(list(range(-1, n_bones - 1)), joints, axes, np.ones(n_bones),
                    np.full(n_bones, radius), [f"bone{i}" for i in range(n_bones)])


def about_axis(pivot, axis, angle):
    """``RigidTransform::about_axis`` (geometry.cpp:7-14): Rodrigues rotation about
    the line through ``pivot``; returns a 3×4 [R | pivot − R·pivot]."""
    n = np.linalg.norm(axis)
    if n < 1e-12:
        raise ValueError("RigidTransform::about_axis: axis must be nonzero")
    k = np.asarray(axis, dtype=np.float64) / n
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    R = np.eye(3) + np.sin(angle) * K + (1.0 - np.cos(angle)) * (K @ K)
    out = np.zeros((3, 4))
    out[:, :3] = R
    out[:, 3] = pivot - R @ pivot
    return out


def compose(a, b):
    """a ∘ b (geometry.hpp:54-56)."""
    out = np.zeros((3, 4))
    out[:, :3] = a[:, :3] @ b[:, :3]
    out[:, 3] = a[:, :3] @ b[:, 3] + a[:, 3]
    return out


def forward_kinematics(skel: Skeleton, angles) -> np.ndarray:
    """``forward_kinematics`` (skeleton.cpp:64-86) → bones [n,3,4] (float64)."""
    skel.validate()
    n = skel.bone_count
    angles = np.asarray(angles, dtype=np.float64)
    if angles.shape[0] != n:
        raise ValueError(f"forward_kinematics: pose has {angles.shape[0]} angles, skeleton expects {n}")
    world = [None] * n

    def resolve(i):
        if world[i] is None:
            local = about_axis(skel.joints[i], skel.axes[i], angles[i])
            p = skel.parents[i]
            world[i] = local if p < 0 else compose(resolve(p), local)
        return world[i]

    for i in range(n):
        resolve(i)
    return np.stack(world)


def apply(T, x):
    return x @ T[:, :3].T + T[:, 3]


def capsules(skel: Skeleton):
    """``CapsuleBody::from_skeleton`` (shape.cpp:21-35): (a[n,3], b[n,3], r[n])."""
    segs = [skel.bone_segment(i) for i in range(skel.bone_count)]
    a = np.stack([s[0] for s in segs])
    b = np.stack([s[1] for s in segs])
    return a, b, skel.radii.copy()


def _bounds(a, b, r):
    lo = np.minimum(a - r[:, None], b - r[:, None]).min(0)
    hi = np.maximum(a + r[:, None], b + r[:, None]).max(0)
    return lo, hi


def padded(lo, hi, frac):
    d = np.linalg.norm(hi - lo)
    return lo - frac * d, hi + frac * d


def canonical_domain(skel: Skeleton):
    """``canonical_domain`` (diff.cpp:128-131): capsule bounds + 10% of their diagonal."""
    a, b, r = capsules(skel)
    return padded(*_bounds(a, b, r), 0.1)


def posed_sampling_box(skel: Skeleton, bones, pad_frac=0.1):
    """``posed_sampling_box`` (diff.cpp:133-137) over ``posed_bounds`` (shape.cpp:110-119)."""
    a, b, r = capsules(skel)
    pa = np.stack([apply(bones[i], a[i]) for i in range(len(r))])
    pb = np.stack([apply(bones[i], b[i]) for i in range(len(r))])
    return padded(*_bounds(pa, pb, r), pad_frac)


def point_segment_distance(p, a, b):
    """``point_segment_distance`` (geometry.cpp:17-23), vectorised over p [m,3]."""
    ab = b - a
    len2 = ab @ ab
    if len2 < 1e-24:
        return np.linalg.norm(p - a, axis=-1)
    t = np.clip(((p - a) @ ab) / len2, 0.0, 1.0)
    return np.linalg.norm(p - (a + t[:, None] * ab), axis=-1)


def vertex_positions(dims, lo, hi):
    """``SkinningVoxelGrid::vertex_position`` (skinning.cpp:77-80), x-fastest [V,3]."""
    nx, ny, nz = dims
    h = (hi - lo) / (np.array(dims) - 1)
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return np.stack([lo[0] + i.ravel() * h[0], lo[1] + j.ravel() * h[1], lo[2] + k.ravel() * h[2]], -1)


def analytic_weight_grid(skel: Skeleton, dims, lo, hi) -> np.ndarray:
    """``analytic_weight_grid`` (fskin_cli.cpp:277-300) → weights [V, n_b] float64."""
    a, b, _ = capsules(skel)
    tau = (0.1 * np.linalg.norm(hi - lo)) ** 2
    x = vertex_positions(dims, lo, hi)
    nb = skel.bone_count
    z = np.full((x.shape[0], nb), -1e6)
    for c in range(nb):  # capsule c belongs to bone c
        d = point_segment_distance(x, a[c], b[c])
        z[:, c] = np.maximum(z[:, c], -d * d / tau)
    z -= z.max(1, keepdims=True)  # softmax_inplace (mlp.cpp:33-37)
    e = np.exp(z)
    return e / e.sum(1, keepdims=True)


def uniform_points(lo, hi, n, rng) -> np.ndarray:
    """Uniform queries in a box (fskin_cli.cpp:629-637)."""
    return lo + rng.random((n, 3)) * (hi - lo)


def ray_points(lo, hi, n, rng, samples=64) -> np.ndarray:
    """Dense ray samples (BASELINE configs[4]: "rays through the posed box, 64 samples per
    ray"): n // samples rays, each from a point on the sphere around the box (radius = the box diagonal)
    towards a uniform point in the box, sampled at `samples` stratified depths (jittered within each
    stratum) over the ray's segment inside the box (slab intersection) — consecutive points are one
    ray's samples, front to back."""
    lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
    n_rays = -(-n // samples)
    c, diag = 0.5 * (lo + hi), np.linalg.norm(hi - lo)
    d = rng.normal(size=(n_rays, 3))
    o = c + diag * d / np.linalg.norm(d, axis=1, keepdims=True)
    t = lo + rng.random((n_rays, 3)) * (hi - lo)
    v = t - o
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    with np.errstate(divide="ignore", invalid="ignore"):
        t0, t1 = (lo - o) / v, (hi - o) / v
    near = np.nanmax(np.minimum(t0, t1), axis=1)
    far = np.nanmin(np.maximum(t0, t1), axis=1)  # the ray hits the box: it aims at a point inside
    u = (np.arange(samples) + rng.random((n_rays, samples))) / samples
    depth = near[:, None] + u * (far - near)[:, None]
    pts = o[:, None, :] + depth[..., None] * v[:, None, :]
    return np.clip(pts.reshape(-1, 3)[:n], lo, hi)


def training_points(skel: Skeleton, bones, n, rng, near_sigma_frac=0.01, pad_frac=0.1):
    """``make_training_frame`` point mix (diff.cpp:148-182): half uniform in the padded
    posed box, half near-surface (area-weighted capsule surface sample moved by its
    bone, + N(0, σ²) with σ = near_sigma_frac·diag)."""
    lo, hi = posed_sampling_box(skel, bones, pad_frac)
    sigma = near_sigma_frac * np.linalg.norm(hi - lo)
    nu = n // 2
    out = np.empty((n, 3))
    out[:nu] = uniform_points(lo, hi, nu, rng)
    a, b, r = capsules(skel)
    L = np.linalg.norm(b - a, axis=1)
    area = 2 * np.pi * r * L + 4 * np.pi * r * r
    m = n - nu
    ci = rng.choice(len(r), size=m, p=area / area.sum())
    side = rng.random(m) * (area[ci]) < 2 * np.pi * r[ci] * L[ci]
    pts = np.empty((m, 3))
    for q in range(m):
        c = ci[q]
        if side[q] and L[c] > 1e-12:
            ax = (b[c] - a[c]) / L[c]
            ref = np.array([1.0, 0, 0]) if abs(ax[0]) < 0.9 else np.array([0, 1.0, 0])
            u = np.cross(ax, ref)
            u /= np.linalg.norm(u)
            v = np.cross(ax, u)
            t, phi = rng.random(), 2 * np.pi * rng.random()
            s = a[c] + t * (b[c] - a[c]) + r[c] * (np.cos(phi) * u + np.sin(phi) * v)
        else:
            d = rng.normal(size=3)
            d /= np.linalg.norm(d)
            ax = (b[c] - a[c]) / L[c] if L[c] > 1e-12 else np.array([0, 0, 1.0])
            s = (b[c] if d @ ax >= 0 else a[c]) + r[c] * d
        pts[q] = apply(bones[c], s)
    out[nu:] = pts + sigma * rng.normal(size=(m, 3))
    return out


@dataclass
class Scene:
    """One deformer workload, all arrays float32 exactly as fed to both paths."""
    dims: tuple
    bbox: np.ndarray        # [6] lo xyz, hi xyz (float32)
    weights: np.ndarray     # [V, nb] float32
    bones: np.ndarray       # [nb, 12] float32 row-major 3×4
    points: np.ndarray      # [N, 3] float32
    angles: np.ndarray
    diag: float             # canonical bbox diagonal (from the float32 bbox)

    @property
    def n_bones(self) -> int:
        return self.bones.shape[0]

    def search_options(self, max_iters=50):
        """``SearchOptions::defaults_for`` (correspondence.cpp:10-17)."""
        return dict(max_iters=max_iters, conv_eps=1e-5 * self.diag, div_eps=0.5 * self.diag,
                    dedup_dist=1e-2 * self.diag)


def make_scene(dims=(32, 32, 32), n_points=10_000, seed=1, pose="random", points="uniform",
               skeleton: Skeleton | None = None) -> Scene:
    """Build a seeded workload. ``pose``: "random" = angles U(−0.5,0.5) (seed), "bench" =
    all 0.4 rad (fskin_cli.cpp:624-625), "rest" = zeros, or an explicit angle array."""
    skel = skeleton or smpl_like_skeleton()
    rng = np.random.default_rng(seed)
    nb = skel.bone_count
    if isinstance(pose, str):
        angles = {"random": lambda: rng.uniform(-0.5, 0.5, nb), "bench": lambda: np.full(nb, 0.4),
                  "rest": lambda: np.zeros(nb)}[pose]()
    else:
        angles = np.asarray(pose, dtype=np.float64)
    bones = forward_kinematics(skel, angles)
    lo, hi = canonical_domain(skel)
    bbox32 = np.concatenate([lo, hi]).astype(np.float32)
    lo32, hi32 = bbox32[:3].astype(np.float64), bbox32[3:].astype(np.float64)
    w = analytic_weight_grid(skel, dims, lo32, hi32).astype(np.float32)
    if points == "uniform":
        plo, phi = posed_sampling_box(skel, bones, 0.1)
        x = uniform_points(plo, phi, n_points, rng)
    elif points == "training":
        x = training_points(skel, bones, n_points, rng)
    elif points == "rays":
        plo, phi = posed_sampling_box(skel, bones, 0.1)
        x = ray_points(plo, phi, n_points, rng)
    else:
        raise ValueError(points)
    return Scene(tuple(dims), bbox32, np.ascontiguousarray(w),
                 np.ascontiguousarray(bones.reshape(nb, 12).astype(np.float32)),
                 np.ascontiguousarray(x.astype(np.float32)), angles,
                 float(np.linalg.norm(hi32 - lo32)))
