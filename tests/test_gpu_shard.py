"""GPU (>= 2 devices): the row-sharded single-instance projection (SURVEY §8e,
tp_solver_set_comm) over 2 ranks returns bitwise the single-GPU solve: every
rank's state equals the unsharded state after 12 iterations, and the traces,
edges and weights agree exactly (tools/shard_check.py under torchrun)."""
import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_projection_bitwise_two_ranks():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tools", "shard_check.py"), "--size", "512", "--iters", "12"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    line = [l for l in p.stdout.splitlines() if l.startswith("{")][-1]
    r = json.loads(line)
    assert r["ranks_agree"] and r["state_equal_to_single_gpu"]
    assert r["trace_equal"] and r["edges_equal"] and r["weights_equal"]
