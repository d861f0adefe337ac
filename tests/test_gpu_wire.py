"""One cmd_deform frame from files to file on the GPU (fsk_deform_files: SKNV + .bin in,
correspondence dump out) — byte-identical to dumping fsk_deform_host's CorrespondenceSets."""
import numpy as np
import pytest
import torch

from paper_2211_15601_b200 import synthetic as S
from paper_2211_15601_b200.deformer import (SearchOptions, deform_files, write_correspondence_dump, write_points_bin,
                                            write_sknv)

pytestmark = pytest.mark.gpu


def test_deform_files_equals_host_path(deformer, tmp_path):
    sc = S.make_scene((32, 32, 32), 30_000, seed=51, points="training")
    g, p, d1, d2 = (str(tmp_path / f) for f in ("g.sknv", "p.bin", "a.txt", "b.txt"))
    write_sknv(g, sc.dims, sc.bbox, torch.from_numpy(sc.weights))
    write_points_bin(p, torch.from_numpy(sc.points))
    o = sc.search_options(50)
    opts = SearchOptions(50, o["conv_eps"], o["div_eps"], o["dedup_dist"])
    nq, nr = deform_files(deformer, g, torch.from_numpy(sc.bones), p, opts, d1)
    n = sc.points.shape[0]
    offs, roots = torch.empty(n + 1, dtype=torch.int64), torch.empty((n * 24, 16), dtype=torch.float32)
    total = deformer.deform_host(torch.from_numpy(sc.weights), sc.dims, sc.bbox, torch.from_numpy(sc.bones),
                                 torch.from_numpy(sc.points), opts, offs, roots)
    write_correspondence_dump(d2, torch.from_numpy(sc.points), offs, roots[:max(total, 1)])
    assert (nq, nr) == (n, total)
    a, b = open(d1).read(), open(d2).read()
    assert a == b and a.count("\n") == n
