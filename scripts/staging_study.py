"""Would staging a sorted tile's sub-grid in shared memory serve the float32 pass's gathers?
(the north star's shared-memory/TMA idea.)

Trajectories come from the oracle itself: the iterate after k Broyden steps is the oracle's x_c
at max_iters = k for a solve still running at k (correspondence.cpp:97-124 keeps x when it stops
at the cap), so the float32 pass's evaluation points are x_0 = B^-1 x', x_1 .. x_min(iters, 8).
Queries in Morton order, tiles of 128 (the k_search_fast block), C2 scene (200 k × 24, 32^3).

Per evaluation, the cell it gathers: a hit in the thread's register cell cache (same cell as the
solve's previous evaluation) costs no gather. For the rest, the fraction inside a box staged
per block is reported for two boxes a CTA could stage:
  (a) per (tile, bone): the vertex box of the tile's init cells (+ margin), staged before each bone
      (a CTA barrier per bone);
  (b) per tile: the vertex box of the tile's converged roots over all bones (an oracle — the
      best a once-per-tile box could do), capped at the shared memory a CTA can hold.
Writes profiles/r02_staging_study.log.
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2211_15601_b200 import synthetic as S  # noqa: E402

TILE, M, CAP32 = 128, 40960, 8


def main():
    sc = S.make_scene((32, 32, 32), 200_000, seed=1)
    nb = sc.n_bones
    p = sc.points.astype(np.float64)
    lo, hi = p.min(0), p.max(0)
    qz = np.clip(((p - lo) / (hi - lo) * 1023).astype(np.int64), 0, 1023)

    def spread(v):
        r = np.zeros_like(v)
        for b in range(10):
            r |= ((v >> b) & 1) << (3 * b)
        return r

    order = np.argsort(spread(qz[:, 0]) | spread(qz[:, 1]) << 1 | spread(qz[:, 2]) << 2, kind="stable")
    pts = sc.points[order][:M].astype(np.float32)
    o = sc.search_options(50)
    full = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, pts, workers=16, **o)
    iters = full["iters"]
    dims = np.array(sc.dims)
    blo, bhi = sc.bbox[:3], sc.bbox[3:]
    scale = (dims - 1) / (bhi - blo)

    def cell(x):
        return np.clip(np.floor((x - blo) * scale).astype(np.int64), 0, dims - 2)

    B = sc.bones.reshape(nb, 3, 4).astype(np.float64)
    traj = np.empty((CAP32 + 1, M, nb, 3))
    for b in range(nb):
        traj[0, :, b] = (pts.astype(np.float64) - B[b, :, 3]) @ np.linalg.inv(B[b, :, :3]).T
    for k in range(1, CAP32 + 1):
        ok = dict(o, max_iters=k)
        traj[k] = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, pts, workers=16, **ok)["x_c"]
    n_eval = np.minimum(iters, CAP32) + 1  # evaluations of the float32 pass per solve
    cells = cell(traj)  # [k, M, nb, 3]
    k_idx = np.arange(CAP32 + 1)[:, None, None]
    valid = k_idx < n_eval[None]
    same = np.zeros_like(valid)
    same[1:] = (cells[1:] == cells[:-1]).all(-1) & valid[1:]
    gathers = valid & ~same
    print(f"C2 sample {M} queries x {nb} bones, {valid.sum()} float32 evaluations, "
          f"{valid.sum() / (M * nb):.2f} per solve")
    print(f"register-cache hits (same cell as the solve's previous evaluation): "
          f"{same.sum() / valid.sum():.3f} of evaluations, {same[1:].sum() / valid[1:].sum():.3f} of iterations "
          f"(the kernel's own counter on C2: 0.527 of iterations)")

    conv = full["converged"] == 1
    roots = cell(full["x_c"])
    out = []
    for margin in (0, 1, 2):
        ins_a = tot = 0
        vols = []
        for t0 in range(0, M, TILE):
            sl = slice(t0, t0 + TILE)
            for b in range(nb):
                c0 = cells[0, sl, b]
                mn, mx = c0.min(0) - margin, c0.max(0) + 1 + margin
                vols.append(np.prod(mx - mn + 1))
                c = cells[:, sl, b]
                g = gathers[:, sl, b]
                inside = ((c >= mn) & (c + 1 <= mx)).all(-1)
                ins_a += (inside & g).sum()
                tot += g.sum()
        vols = np.array(vols)
        out.append(f"(a) per-bone init box, margin {margin}: {ins_a / tot:.3f} of the gathers inside; box "
                   f"median {np.median(vols):.0f} vertices ({np.median(vols) * 96 / 1024:.0f} KB at 96 B per vertex), "
                   f"p90 {np.percentile(vols, 90):.0f}")
    for cap in (512, 1024, 2048):
        ins_b = tot = 0
        for t0 in range(0, M, TILE):
            sl = slice(t0, t0 + TILE)
            r = roots[sl][conv[sl]]
            g = gathers[:, sl]
            tot += g.sum()
            if len(r) == 0:
                continue
            mn, mx = r.min(0), r.max(0) + 1
            if np.prod(mx - mn + 1) > cap:
                continue
            c = cells[:, sl]
            ins_b += (((c >= mn) & (c + 1 <= mx)).all(-1) & g).sum()
        out.append(f"(b) per-tile roots box (oracle roots), staged when <= {cap} vertices "
                   f"({cap * 96 // 1024} KB): {ins_b / tot:.3f} of the gathers inside")
    for line in out:
        print(line)


if __name__ == "__main__":
    main()
