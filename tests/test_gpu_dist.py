"""GPU: the real multi-process row-sharded path (shard.DistGroup: one
process per rank under torch.distributed.run, CUDA-IPC mapped peer
workspaces, device mailbox exchanges) -- two ranks on the test box's GPU.
The sharded iterate equals the one-GPU iterate up to reduction-order
rounding and every rank holds the same bits."""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_dist_group_two_processes_cuda_ipc(cuda):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, AQP_COMM_TIMEOUT_S="60", CUDA_DEVICE_MAX_CONNECTIONS="32")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "helpers", "dist_shard_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 2, out.stdout[-2000:]
    for d in lines:
        assert d["ranks_identical"], d
        assert d["status"] == "iteration_limit" or d["outer"] == d["single_outer"], d
        assert d["max_dx"] <= 1e-8 * d["scale"] and d["max_dy"] <= 1e-8 * max(1.0, d["scale"]), d
