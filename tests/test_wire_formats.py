"""Wire and disk formats through the C-ABI host helpers: SKNV grids
(skinning.cpp:239-288), .bin points (pointio.cpp:43-62), correspondence dumps
(pointio.cpp:97-117, "%.17g" text). CPU-only: no device is touched."""
import os

import numpy as np
import pytest
import torch

from paper_2211_15601_b200 import build as B
from paper_2211_15601_b200 import synthetic as S

B.build()
from paper_2211_15601_b200.deformer import (FskError, FskInvalidArgument, read_points_bin, read_sknv,  # noqa: E402
                                            write_correspondence_dump, write_points_bin, write_sknv)


def test_sknv_roundtrip_and_layout(tmp_path):
    sc = S.make_scene((5, 4, 3), 10, seed=1)
    p = str(tmp_path / "g.sknv")
    write_sknv(p, sc.dims, sc.bbox, torch.from_numpy(sc.weights))
    raw = open(p, "rb").read()
    assert raw[:4] == b"SKNV" and np.frombuffer(raw[4:24], np.uint32).tolist() == [1, 5, 4, 3, 24]
    assert np.array_equal(np.frombuffer(raw[24:48], np.float32), sc.bbox)
    assert np.array_equal(np.frombuffer(raw[48:], np.float32).reshape(-1, 24), sc.weights)
    dims, bbox, w = read_sknv(p)
    assert dims == (5, 4, 3) and np.array_equal(bbox, sc.bbox) and np.array_equal(w.numpy(), sc.weights)


def test_sknv_errors(tmp_path):
    bad = tmp_path / "bad.sknv"
    bad.write_bytes(b"XXXX" + b"\0" * 40)
    with pytest.raises(FskError, match="not a SKNV grid file"):
        read_sknv(str(bad))
    bad.write_bytes(b"SKNV" + np.array([2, 2, 2, 2, 1], np.uint32).tobytes() + b"\0" * 24)
    with pytest.raises(FskError, match="unsupported SKNV version 2"):
        read_sknv(str(bad))
    hdr = b"SKNV" + np.array([1, 2, 2, 2, 1], np.uint32).tobytes() + np.array([0, 0, 0, 1, 1, 1], np.float32).tobytes()
    bad.write_bytes(hdr + b"\0" * 8)
    with pytest.raises(FskError, match="truncated SKNV payload"):
        read_sknv(str(bad))
    bad.write_bytes(b"SKNV" + np.array([1, 1, 2, 2, 1], np.uint32).tobytes() + b"\0" * 24)
    with pytest.raises(FskInvalidArgument, match="dims must be >= 2 per axis"):
        read_sknv(str(bad))
    with pytest.raises(FskError, match="cannot open grid file"):
        read_sknv(str(tmp_path / "missing.sknv"))


def test_points_bin_roundtrip_and_errors(tmp_path):
    x = np.random.default_rng(0).normal(size=(1001, 3)).astype(np.float32)
    p = str(tmp_path / "p.bin")
    write_points_bin(p, torch.from_numpy(x))
    assert os.path.getsize(p) == 1001 * 12
    assert np.array_equal(read_points_bin(p).numpy(), x)
    (tmp_path / "odd.bin").write_bytes(b"\0" * 13)
    with pytest.raises(FskError, match="size 13 is not a whole number of f32 triples"):
        read_points_bin(str(tmp_path / "odd.bin"))


def _py_dump(q, offs, roots):
    lines = []
    for i in range(len(q)):
        s = "%.17g %.17g %.17g %d" % (*[float(v) for v in q[i]], offs[i + 1] - offs[i])
        for r in range(offs[i], offs[i + 1]):
            R = roots[r]
            bone, it = R[13:15].view(np.int32)
            s += " %.17g %.17g %.17g %.17g %d %d" % (float(R[0]), float(R[1]), float(R[2]), float(R[3]), bone, it)
        lines.append(s + "\n")
    return "".join(lines)


@pytest.mark.parametrize("threads", [1, 3, 0])
def test_correspondence_dump_matches_printf(tmp_path, threads):
    rng = np.random.default_rng(threads)
    n = 2000
    q = rng.normal(size=(n, 3)).astype(np.float32)
    q[0] = [0.0, -0.0, 1e-30]
    q[1] = [123456.789, -1e-7, 3.0]
    counts = rng.integers(0, 4, n)
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    roots = rng.normal(size=(offs[-1], 16)).astype(np.float32)
    roots[:, 13:16] = np.stack([rng.integers(0, 24, offs[-1]), rng.integers(0, 51, offs[-1]),
                                np.zeros(offs[-1], int)], 1).astype(np.int32).view(np.float32)
    p = str(tmp_path / "c.txt")
    write_correspondence_dump(p, torch.from_numpy(q), torch.from_numpy(offs), torch.from_numpy(roots), threads)
    assert open(p).read() == _py_dump(q, offs, roots)
