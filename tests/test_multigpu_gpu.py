"""Multi-GPU parity (one process per GPU through torchrun): runs
scripts/mgpu_check.py on every visible GPU (at most 4) for both exchange
paths -- the fused peer-memory (P2P) path and the NCCL baseline -- with
serving ranks placed by overlap (the bench's placement), and the P2P path
with the reference's rank order.  Skipped on
a single-GPU box; the CPU side of the N>1 logic is covered by
tests/test_multirank_cpu.py."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("mode", ["p2p", "nccl", "p2p_rank"])
def test_mgpu_check(mode):
    """p2p_rank: serving rank g on GPU g (WS_PLACE_RANK)."""
    n = min(torch.cuda.device_count(), 4)
    if n < 2:
        pytest.skip("needs at least 2 GPUs")
    env = dict(os.environ, WSYNC_EXCHANGE=mode.split("_")[0])
    if mode == "p2p_rank":
        env["WSYNC_CHECK_PLACEMENT"] = "rank"
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
                        "--master-port", str(_port()), os.path.join(ROOT, "scripts", "mgpu_check.py")],
                       capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert len(lines) == n and all(l["ok"] for l in lines), lines
