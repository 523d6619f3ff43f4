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
@pytest.mark.parametrize("p2p,ll", [("1", "1"), ("1", "0"), ("0", "1")],
                         ids=["fused_peer_ll", "fused_peer_fenced", "nccl"])
def test_sharded_equals_replica(p2p, ll):
    """fused_peer_ll: the default flag-in-data lines (REC_P2P_LL=1) for the asynchronous
    synthetic chains; fused_peer_fenced: pooled vectors stored straight into the owner's X
    behind the per-CTA system-scope fence (REC_P2P_LL=0)."""
    import __graft_entry__
    __graft_entry__.build()
    n = min(_ngpus(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "295" + p2p + ll,
           os.path.join(ROOT, "scripts", "shard_check.py"), "--iters", "5"]
    env = dict(os.environ, REC_P2P=p2p, REC_P2P_LL=ll, REC_VERBOSE="1")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    line = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert p.returncode == 0 and line, p.stdout[-3000:] + p.stderr[-3000:]
    res = json.loads(line[-1])
    assert res["ok"], res
    fused = "over peer memory" in p.stderr
    assert fused == (p2p == "1"), p.stderr[-2000:]


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
def test_bench_line_on_two_gpus():
    """The driver's scaling runs launch `bench.py --gpus N` under torch.distributed.run: replica
    models then carry a communicator (all-rank serving percentiles) and every measurement pass
    must accept them; the rank-0 line reports n_gpus = 2 with library-gathered p95s."""
    import __graft_entry__
    __graft_entry__.build()
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3", "--step-batches", "16",
           "--per-model", "rmc3", "--pm-steps", "2", "--pm-step-batches", "16", "--pm-sla", "0",
           "--sla-queries", "3000", "--max-batch-search", "256", "--mlp-batch", "0", "--e2e-steps", "1",
           "--caller-batches", "2", "--roofline-steps", "8", "--sls-batches", "8", "--no-cpu-baseline"]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    line = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert p.returncode == 0 and len(line) == 1, p.stdout[-2000:] + p.stderr[-3000:]
    d = json.loads(line[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "weak"
    assert d["sla"]["lambda_star_qps"] > 0
    assert all(pr.get("p95_from") == "library (all ranks)" for pr in d["sla"]["probes_at_best"] or [])


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs")
def test_missing_peer_times_out_with_error():
    """A sharded batch that a peer never joins: every cross-GPU wait of the chain (hint flags,
    flag-in-data lines, CTR flags) is bounded by REC_P2P_TIMEOUT_S and rec_sync reports
    REC_E_NCCL; the CUDA context keeps working (no trap)."""
    import __graft_entry__
    __graft_entry__.build()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29571",
           os.path.join(ROOT, "scripts", "p2p_timeout_check.py")]
    env = dict(os.environ, REC_P2P_TIMEOUT_S="2")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    line = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert p.returncode == 0 and line, p.stdout[-3000:] + p.stderr[-3000:]
    res = json.loads(line[-1])
    assert res["ok"] and res["lone_batch_status"] == -6, res
