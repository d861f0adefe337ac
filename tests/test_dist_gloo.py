"""The N>1 host path on CPU: world_size-2 gloo process group, compute injected from the
oracle (the checker), verifying that sharded + gathered results equal the single-process
run bitwise (SPEC.md:573 determinism across worker counts) and that the all-reduced
backward equals the full-batch grid VJP."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_15601_b200 import dist as fdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_is_parallel_for_partition():
    n = 1001
    for w in (1, 2, 3, 8):
        parts = [fdist.shard_range(n, r, w) for r in range(w)]
        assert parts[0][0] == 0 and parts[-1][1] == n
        assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
        assert parts == [(n * r // w, n * (r + 1) // w) for r in range(w)]


def _worker(rank, world, port, q):
    import oracle
    from paper_2211_15601_b200 import synthetic as S
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = S.make_scene((16, 16, 16), 301, seed=4)
        w = torch.from_numpy(sc.weights.copy()) if rank == 0 else torch.zeros_like(torch.from_numpy(sc.weights))
        B = torch.from_numpy(sc.bones.copy()) if rank == 0 else torch.zeros_like(torch.from_numpy(sc.bones))
        fdist.broadcast_inputs([w, B], src=0)
        assert torch.equal(w, torch.from_numpy(sc.weights)) and torch.equal(B, torch.from_numpy(sc.bones))
        opts = sc.search_options(30)

        def search_fn(x):
            r = oracle.batch_search(w.numpy(), sc.dims, sc.bbox, B.numpy(), x.numpy(), workers=1, **opts)
            return {k: torch.from_numpy(v) for k, v in r.items()}

        res, (a, b) = fdist.sharded_forward(torch.from_numpy(sc.points), search_fn, gather=True)
        n = sc.points.shape[0]
        v = torch.from_numpy(np.random.default_rng(0).normal(size=(n, 3)) / n)
        keep = res["keep"].numpy()
        sel = np.where(keep.any(1), np.argmax(keep, 1), -1).astype(np.int32)

        def local_grad():
            ls = sel[a:b]
            idx = np.arange(b - a)
            xs = res["x_c"].numpy()[a:b][idx, np.maximum(ls, 0)]
            J = res["jinv"].numpy()[a:b][idx, np.maximum(ls, 0)]
            gT, _ = oracle.grid_vjp(sc.dims, sc.bbox, B.numpy(), xs, J, v.numpy()[a:b], sel=ls)
            return torch.from_numpy(gT)

        gT, _ = fdist.sharded_backward(local_grad)
        if rank == 0:
            q.put((({k: t.numpy() for k, t in res.items()}), gT.numpy(), sel, v.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_forward_and_backward_match_single_process():
    import oracle
    from paper_2211_15601_b200 import synthetic as S
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res, gT, sel, v = q.get(timeout=240)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    sc = S.make_scene((16, 16, 16), 301, seed=4)
    full = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=1, **sc.search_options(30))
    for k in full:
        np.testing.assert_array_equal(res[k], full[k])  # bitwise: sharding never changes a solve
    n = sc.points.shape[0]
    xs = full["x_c"][np.arange(n), np.maximum(sel, 0)]
    J = full["jinv"][np.arange(n), np.maximum(sel, 0)]
    rT, _ = oracle.grid_vjp(sc.dims, sc.bbox, sc.bones, xs, J, v, sel=sel)
    np.testing.assert_allclose(gT, rT, rtol=0, atol=1e-14)
