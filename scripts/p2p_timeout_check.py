"""Bounded cross-GPU waits (include/rec.h rec_sync): a table-wise sharded batch
that a peer never joins must come back as REC_E_NCCL within the configured timeout instead of
hanging the stream or trapping the CUDA context.

Both ranks first run one batch together (sanity, CTRs bit-exact vs a replica); then rank 0
submits a batch alone.  Its chain waits for rank 1's hint flags (k_p2p_wait), spins on the
flag-in-data lines rank 1 never writes (k_p2p_ll_unpack), and waits for rank 1's CTR flags;
each wait gives up after REC_P2P_TIMEOUT_S and sets the error flag.  Rank 0 checks that
rec_sync raises REC_E_NCCL after about the timeout and that its CUDA context still runs work.
usage: REC_P2P_TIMEOUT_S=2 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/p2p_timeout_check.py
Prints one JSON line on rank 0; exit code 1 on failure.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    import workloads as W
    from paper_2203_07424_b200 import RecModel, RecError, nccl_unique_id, REC_SHARD_TABLE
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    timeout_s = float(os.environ.get("REC_P2P_TIMEOUT_S", "60"))
    t = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0)
    cfg = W.small_variant(W.RMC2, 4096)
    m = RecModel(cfg, seed=1, max_batch=1024, streams=2, device=local, shard=REC_SHARD_TABLE,
                 rank=rank, world=world, nccl_id=bytes(t.cpu().numpy()))
    rep = RecModel(cfg, seed=1, max_batch=1024, device=local)
    res = {"world": world, "timeout_s": timeout_s}
    segs = W.random_segments(300, seed=9)
    out = torch.zeros(300, device="cuda")
    ref = torch.zeros(300, device="cuda")
    m.rec_synth_query_async(0, segs, out)                  # every rank: a normal batch
    m.rec_sync(0)
    rep.rec_synth_query_async(0, segs, ref)
    rep.rec_sync(0)
    res["joint_batch_bit_exact"] = bool(torch.equal(out, ref))
    dist.barrier()
    if rank == 0:                                          # rank 0 alone: the peer never joins
        t0 = time.perf_counter()
        code = None
        try:
            m.rec_synth_query_async(1, segs, out)
            m.rec_sync(1)
        except RecError as e:
            code = e.status
        res["lone_batch_status"] = code
        res["lone_batch_wall_s"] = round(time.perf_counter() - t0, 2)
        res["context_alive"] = float(torch.ones(4, device="cuda").sum().item()) == 4.0
    dist.barrier()
    m.close()
    rep.close()
    ok = res["joint_batch_bit_exact"]
    if rank == 0:
        ok = ok and res["lone_batch_status"] == -6 and res["context_alive"] and \
            res["lone_batch_wall_s"] < 6 * timeout_s + 30
        res["ok"] = bool(ok)
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
