"""World-size-2 gloo tests of the multi-GPU host logic (CPU only).

* shard plans of all ranks (C++ rec_shard_plan) partition tables / rows / item blocks
  exactly (table-wise and row-wise);
* replica serving: the bench harness's trace partition (query q -> rank q mod G) and the
  rank-0 latency gather give the same p95 as one process replaying the whole trace's
  per-rank shares (oracle virtual clock)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # surfaced by the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world=2, port=29601):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return out


def _plans(rank, world):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2203_07424_b200 import rec_shard_plan, REC_SHARD_TABLE, REC_SHARD_ROW
    res = {}
    for name, rows, shard, B in (("table", [1000] * 40, REC_SHARD_TABLE, 1025),
                                 ("row", [1_000_003] * 10, REC_SHARD_ROW, 7)):
        p = rec_shard_plan(rows, world, rank, shard, B)
        t = torch.tensor([p["t0"], p["t_local"], p["row_lo"], p["row_hi"], p["item0"], p["items"]],
                         dtype=torch.int64)
        g = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(g, t)
        res[name] = [x.tolist() for x in g]
    return res


def test_shard_plans_partition_gloo():
    import __graft_entry__
    __graft_entry__.build()
    out = _spawn(_plans)
    assert not isinstance(out[0], str), out
    tab = out[0]["table"]
    assert out[1]["table"] == tab
    tables = sorted(t for p in tab for t in range(p[0], p[0] + p[1]))
    assert tables == list(range(40))
    items = sorted(i for p in tab for i in range(p[4], p[4] + p[5]))
    assert items == list(range(1025))
    row = out[0]["row"]
    assert [p[1] for p in row] == [10, 10]
    spans = sorted((p[2], p[3]) for p in row)
    assert spans[0][0] == 0 and spans[-1][1] == 1_000_003 and spans[0][1] == spans[1][0]
    assert sorted(i for p in row for i in range(p[4], p[4] + p[5])) == list(range(7))


def _replica_p95(rank, world):
    import sys
    sys.path.insert(0, ROOT)
    from harness import sla
    from oracle import serving as sv
    tr = W.poisson_trace(20000.0, 400, seed=5)
    mine = sla.rank_share(tr, world, rank)
    r = sv.replay_virtual(mine, 2, 256, 20000.0, 30.0)
    lat = sla.gather_latencies(r.latency_s * 1e3, world, rank, dist)
    return None if lat is None else sorted(lat.tolist())


def test_replica_dispatch_and_latency_gather_gloo():
    out = _spawn(_replica_p95, port=29611)
    assert not isinstance(out[0], str), out
    from harness import sla
    from oracle import serving as sv
    tr = W.poisson_trace(20000.0, 400, seed=5)
    parts = [sla.rank_share(tr, 2, r) for r in range(2)]
    assert sorted(np.concatenate([p["qid"] for p in parts]).tolist()) == list(range(400))
    exp = np.concatenate([sv.replay_virtual(p, 2, 256, 20000.0, 30.0).latency_s * 1e3 for p in parts])
    assert out[0] == sorted(exp.tolist())
    assert out[1] is None
