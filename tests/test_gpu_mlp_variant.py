"""MLP-variant search (SearchVariant::Mlp) on the GPU against the f64
oracle restatement, and the SPEC's variant-equivalence criterion: roots of the
MLP variant vs the voxel variant on a grid distilled from the same network."""
import numpy as np
import pytest
import torch

import oracle
from paper_2211_15601_b200 import synthetic as S
from paper_2211_15601_b200.deformer import SearchOptions

pytestmark = pytest.mark.gpu
SKIN = [3, 64, 64, 64, 24]


def _opts(sc, mi=50):
    o = sc.search_options(mi)
    return o, SearchOptions(mi, o["conv_eps"], o["div_eps"], o["dedup_dist"])


def _net(sc, seed, head_scale):
    """A skinning network whose input is conditioned on the canonical box like
    SkinningMlp(n_b, seed, domain) (skinning.cpp:19-23: W0 /= half extent, b0 -= W0·center)."""
    th = oracle.mlp_init(SKIN, seed, head_scale)
    lo, hi = sc.bbox[:3].astype(float), sc.bbox[3:].astype(float)
    c, h = 0.5 * (lo + hi), 0.5 * (hi - lo)
    W0 = th[:192].reshape(3, 64).T / h  # column-major (64 x 3)
    th[:192] = W0.T.reshape(-1)
    th[192:256] -= W0 @ c
    return th.astype(np.float32)


def test_mlp_variant_matches_oracle(deformer):
    sc = S.make_scene((32, 32, 32), 1500, seed=41, points="training")
    th = _net(sc, 3, 0.5)
    o, so = _opts(sc)
    g = deformer.batch_search_mlp(torch.from_numpy(th).cuda(), SKIN, torch.from_numpy(sc.bones).cuda(),
                                  torch.from_numpy(sc.points).cuda(), so)
    g = {k: v.cpu().numpy() for k, v in g.items() if v is not None}
    r = oracle.batch_search_mlp(th, SKIN, sc.bones, sc.points, **o)
    agree = (g["converged"] == r["converged"]).mean()
    both = (g["converged"] == 1) & (r["converged"] == 1)
    dx = np.abs(g["x_c"] - r["x_c"]).max(-1)[both]
    keep_agree = (g["keep"] == r["keep"]).mean()
    print(f"\nmlp variant: converged {r['converged'].mean():.3f}, mask agreement {agree:.6f}, keep {keep_agree:.6f}, "
          f"|dx| p50 {np.median(dx):.1e} p99.9 {np.percentile(dx, 99.9):.1e} max {dx.max():.1e}")
    # float32 trajectories through a float32 network: no float64 escalation on this path
    assert agree >= 0.9999 and keep_agree >= 0.9999
    assert dx.max() <= 1e-4


def _match_sets(xa, ka, xb, kb, tol):
    """Per query: the kept root sets match one-to-one within tol (greedy)."""
    n = ka.shape[0]
    ok = np.zeros(n, bool)
    for q in range(n):
        A, B = xa[q][ka[q] == 1], xb[q][kb[q] == 1]
        if len(A) != len(B):
            continue
        used = np.zeros(len(B), bool)
        good = True
        for a in A:
            d = np.linalg.norm(B - a, axis=1)
            d[used] = np.inf
            j = int(np.argmin(d)) if len(B) else -1
            if j < 0 or d[j] > tol:
                good = False
                break
            used[j] = True
        ok[q] = good
    return ok


@pytest.mark.parametrize("head_scale", [0.05, 0.3])
def test_variant_equivalence_spec(deformer, head_scale):
    """SPEC.md:567 (acceptance 3): MLP-variant and voxel-variant (grid distilled at 64x64x16
    from the same network) root sets match one-to-one within 1e-2·diag on >= 99 % of queries,
    and the match rate at 128x128x32 is at least the rate at 32x32x8 (Table 3 direction).
    Networks: SkinningMlp's own init (head scaled by 0.05, skinning.cpp:10-17) and a sharper
    head (0.3, reported, direction asserted), input conditioned on the canonical box (:19-23)."""
    sc = S.make_scene((64, 64, 16), 10_000, seed=42)
    th = _net(sc, 5, head_scale)
    tht = torch.from_numpy(th).cuda()
    o, so = _opts(sc)
    B, x = torch.from_numpy(sc.bones).cuda(), torch.from_numpy(sc.points).cuda()
    m = deformer.batch_search_mlp(tht, SKIN, B, x, so)
    xm, km = m["x_c"].cpu().numpy(), m["keep"].cpu().numpy()
    rate = {}
    for dims in ((32, 32, 8), (64, 64, 16), (128, 128, 32)):
        w = deformer.distill(tht, SKIN, dims, sc.bbox)
        tg = deformer.precompute_transform_grid(w, dims, sc.bbox, B)
        v = deformer.batch_search(tg, dims, sc.bbox, B, x, so)
        rate[dims] = _match_sets(xm, km, v["x_c"].cpu().numpy(), v["keep"].cpu().numpy(), 1e-2 * sc.diag).mean()
    print(f"\nvariant equivalence (head scale {head_scale}, {km.sum(1).mean():.2f} roots/query): {rate}")
    if head_scale == 0.05:  # the reference's SkinningMlp init: the SPEC's >= 99 % bar
        assert rate[(64, 64, 16)] >= 0.99
    assert rate[(128, 128, 32)] >= rate[(32, 32, 8)]
