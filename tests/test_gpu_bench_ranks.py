"""The multi-rank bench step (torchrun, one process per GPU): per-frame NCCL broadcast of the pose,
per-rank point shards, all-reduced dL/dT in the training shape, max-over-ranks timing. A one-GPU box
cannot run NCCL ranks side by side, so this checks the step's logic with FSK_BENCH_SHARED_GPU=1:
both ranks on cuda:0 over the host-side gloo backend (no rank's kernel waits on another's)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("extra", [[], ["--backward", "--poses", "2", "--no-e2e"],
                                   ["--poses", "3", "--grid", "64,64,64", "--no-e2e"],      # C4 shape: staged poses
                                   ["--grid", "128,128,32", "--no-e2e"]])                   # C5 shape: ray samples
def test_two_rank_bench_step(extra):
    env = dict(os.environ, FSK_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), "bench.py", "--gpus", "2",
           "--points", "20000", "--steps", "2", "--warmup", "3", "--no-mlp", "--no-cpu-baseline", *extra]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 prints the one line
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert "broadcast" in d["config"]["parallelism"]
    if "--backward" in extra:
        assert "all-reduce" in d["config"]["parallelism"]
    if "--poses" in extra and "--backward" not in extra:
        assert d["pipeline"]["poses_staged"]
    if "128,128,32" in extra:
        assert "rays" in d["config"]["workload"]
