"""Multi-GPU sharding parity (needs >= 2 GPUs; skipped otherwise).

Runs scripts/shard_check.py under torchrun: table-wise (all-to-all) and row-wise
(reduce-scatter) sharded CTRs must equal the replica CTRs bit for bit (int8-exact values)
and the CPU oracle within 2e-2 — once with the exchange fused into the SLS kernel (peer
stores over NVLink, REC_P2P default) and once through NCCL collectives (REC_P2P=0)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("p2p", ["1", "0"], ids=["fused_peer", "nccl"])
def test_sharded_equals_replica(p2p):
    import __graft_entry__
    __graft_entry__.build()
    n = min(_ngpus(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "2953" + p2p,
           os.path.join(ROOT, "scripts", "shard_check.py"), "--iters", "5"]
    env = dict(os.environ, REC_P2P=p2p, REC_VERBOSE="1")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    line = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert p.returncode == 0 and line, p.stdout[-3000:] + p.stderr[-3000:]
    res = json.loads(line[-1])
    assert res["ok"], res
    fused = "over peer memory" in p.stderr
    assert fused == (p2p == "1"), p.stderr[-2000:]
