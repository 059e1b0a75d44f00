"""bench.py's population-sharded mode end to end: two ranks (torchrun, gloo,
both on cuda:0 -- the single-GPU stand-in for NCCL on a multi-GPU box) run
one sharded population and rank 0 prints the bench line."""

import json
import os
import socket
import subprocess
import sys

import pytest

from gpu_util import needs_gpu

pytestmark = [pytest.mark.gpu, needs_gpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_shard_mode_two_ranks():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, HARL_DIST_BACKEND="gloo")
    p = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
         "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
         "--master-port", str(port), os.path.join(ROOT, "bench.py"),
         "--gpus", "2", "--steps", "2", "--warmup", "1", "--population",
         "1024", "--no-cpu-baseline"],
        cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-3000:]
    line = json.loads([ln for ln in p.stdout.splitlines()
                       if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert "sharded over 2 GPUs" in line["config"]["parallelism"]
    # 2048 tracks x 40 visits per episode over both ranks
    assert line["value"] > 0 and line["ms_per_step"] > 0
    assert line["e2e"]["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0
