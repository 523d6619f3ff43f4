"""Multi-GPU embedding sharding check + timing (torchrun, one process per GPU).

For table-wise (RMC2 shapes, 40 tables) and row-wise (RMC1 shapes, 10 tables) sharding:
  * every rank builds the sharded model and a full replica, runs rec_query on the same
    global batch, and checks sharded CTR == replica CTR bit for bit (int8-exact values);
  * rank 0 checks the CTRs against the CPU oracle (2e-2);
  * per-batch latency of the sharded query vs the replica query is timed (CUDA events,
    max over ranks) at B = 1024 on full-size tables.
usage: torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/shard_check.py [--full]
Prints one JSON line on rank 0; exit code 1 on any mismatch.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def async_checks(cfg, rank, world, local, bcast_id, rep):
    """Table-wise sharding over peer memory, asynchronous: several global batches
    in flight on several stream slots (device-synthesised inputs, and caller inputs through
    rec_query_async), and rec_serve with the deterministic global dispatcher - every CTR must
    equal the replica's bits."""
    import torch
    import workloads as W
    from paper_2203_07424_b200 import RecModel, REC_SHARD_TABLE
    res = {}
    m = RecModel(cfg, seed=1, max_batch=1024, streams=4, device=local, shard=REC_SHARD_TABLE,
                 rank=rank, world=world, nccl_id=bcast_id())
    batches = [W.random_segments(b, seed=500 + k) for k, b in enumerate((1024, 1, 333, 700, 1000, 5, 1024, 64))]
    outs = [torch.zeros(int(sg[:, 2].sum()), device="cuda") for sg in batches]
    for k, sg in enumerate(batches):                     # 8 batches round-robin on 4 slots
        m.rec_synth_query_async(k % 4, sg, outs[k])
    for s in range(4):
        m.rec_sync(s)
    good = True
    for k, sg in enumerate(batches):
        ref = torch.zeros(outs[k].numel(), device="cuda")
        rep.rec_synth_query_async(0, sg, ref)
        rep.rec_sync(0)
        good &= bool(torch.equal(ref, outs[k]))
    res["async_synth_bit_exact_vs_replica"] = good
    good = True
    for k, sg in enumerate(batches[:4]):                 # caller inputs, asynchronous
        ind, off, dense = rep.rec_gen_batch(sg)
        B = dense.shape[0]
        dv, iv, ov = (torch.from_numpy(x).cuda() for x in (dense, ind, off))
        cv = torch.zeros(B, device="cuda")
        m.rec_query_async(k % 4, dv, iv, ov, int(off[-1]), B, cv)
        m.rec_sync(k % 4)
        good &= bool(torch.equal(cv, outs[k]))
    res["async_caller_bit_exact_vs_replica"] = good
    tr = W.poisson_trace(20000.0, 600, seed=13)
    r = m.rec_serve(tr, 50.0, streams=4, max_batch=1024, want_ctr=True)
    rr = rep.rec_serve(tr, 50.0, streams=1, max_batch=1024, want_ctr=True)
    res["serve_all_completed"] = bool(r["completed"] == len(tr))
    res["serve_ctr_bit_exact_vs_replica"] = bool(np.array_equal(r["ctr"], rr["ctr"]))
    res["info_p95_ms"] = round(r["p95_ms"], 3)
    res["info_batches"] = int(r["batches"])
    m.close()
    return res


def main():
    import torch
    import torch.distributed as dist
    import workloads as W
    from paper_2203_07424_b200 import RecModel, nccl_unique_id, REC_SHARD_TABLE, REC_SHARD_ROW

    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true", help="also time full-size (1M-row) tables")
    ap.add_argument("--iters", type=int, default=50)
    a = ap.parse_args()
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def bcast_id():
        t = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(t, 0)
        return bytes(t.cpu().numpy())

    out = {"world": world, "checks": {}, "timing_us": {}}
    ok = True
    cases = [("table_rmc2", W.small_variant(W.RMC2, 4096), REC_SHARD_TABLE, 333),
             ("row_rmc1", W.small_variant(W.RMC1, 20000), REC_SHARD_ROW, 257)]
    if a.full:
        cases += [("table_rmc2_full", W.RMC2, REC_SHARD_TABLE, 1024),
                  ("row_rmc1_full", W.RMC1, REC_SHARD_ROW, 1024)]
    for name, cfg, shard, B in cases:
        if shard == REC_SHARD_TABLE and cfg.num_tables % world:
            continue
        rep = RecModel(cfg, seed=1, max_batch=max(B, 1024), device=local)
        shm = RecModel(cfg, seed=1, max_batch=max(B, 1024), device=local, shard=shard, rank=rank,
                       world=world, nccl_id=bcast_id())
        segs = W.random_segments(B, seed=77)
        ind, off, dense = rep.rec_gen_batch(segs)
        c_rep = np.zeros(B, np.float32)
        c_sh = np.zeros(B, np.float32)
        rep.rec_query(dense, ind, off, B, c_rep)
        shm.rec_query(dense, ind, off, B, c_sh)
        same = bool(np.array_equal(c_rep, c_sh))
        ok &= same
        chk = {"bit_exact_vs_replica": same}
        if rank == 0 and not name.endswith("_full"):
            from oracle import forward as fw, gen
            oi, oo, od = gen.gen_batch(cfg, 1, segs)
            exp = fw.forward(cfg, 1, od, oi, oo)
            err = float(np.abs(c_sh - exp).max())
            chk["max_abs_err_vs_oracle"] = err
            ok &= err <= 2e-2
        out["checks"][name] = chk
        # timing: synchronous queries on device-resident inputs
        dv, iv, ov = (torch.from_numpy(x).cuda() for x in (dense, ind, off))
        cv = torch.zeros(B, device="cuda")
        res = {}
        for tag, mdl in (("replica", rep), ("sharded", shm)):
            for _ in range(5):
                mdl.rec_query(dv, iv, ov, B, cv)
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            for _ in range(a.iters):
                mdl.rec_query(dv, iv, ov, B, cv)
            torch.cuda.synchronize()
            us = torch.tensor([1e6 * (time.perf_counter() - t0) / a.iters], device="cuda")
            dist.all_reduce(us, op=dist.ReduceOp.MAX)
            res[tag] = round(float(us), 1)
        out["timing_us"][name] = res
        if shard == REC_SHARD_TABLE and name == "table_rmc2" and os.environ.get("REC_P2P", "1") != "0":
            chk.update(async_checks(cfg, rank, world, local, bcast_id, rep))
            ok &= all(v for k, v in chk.items() if k.startswith("async") or k.startswith("serve"))
        shm.close()
        rep.close()
    # replicas with a communicator: rec_serve's percentiles cover every rank's queries (C4)
    cfg = W.small_variant(W.RMC1, 20000)
    rm = RecModel(cfg, seed=1, max_batch=1024, streams=4, device=local, rank=rank, world=world,
                  nccl_id=bcast_id())
    tr = W.poisson_trace(40000.0, 4000, seed=17)
    mine = tr[tr["qid"] % world == rank]
    r = rm.rec_serve(mine, 20.0, 4, 1024, warmup_frac=0.1)
    arr = mine["arrival_s"]
    w_end = arr[0] + 0.1 * (arr[-1] - arr[0])
    parts = [None] * world
    dist.all_gather_object(parts, r["latency_ms"][arr >= w_end])
    lat = np.sort(np.concatenate(parts))
    p95 = float(lat[max((95 * lat.size + 99) // 100, 1) - 1])
    same = bool(r["ranks"] == world and abs(r["p95_ms"] - p95) < 1e-9 and r["completed"] == len(tr))
    out["checks"]["replica_serve_global_p95"] = {"ok": same, "p95_ms": r["p95_ms"], "ranks": r["ranks"]}
    ok &= same
    rm.close()
    okt = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    out["ok"] = bool(okt.item())
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if out["ok"] else 1)


if __name__ == "__main__":
    main()
