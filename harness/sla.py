"""SLA-bounded QPS measurement (S5) across replica GPUs: trace partition (q mod G), rank-0
latency gather (C4), nearest-rank p95, lambda* by geometric bracketing + bisection
 with rec_serve (real clock) as the measurement."""
import numpy as np

import workloads as W


def rank_share(trace: np.ndarray, world: int, rank: int) -> np.ndarray:
    """Replica dispatch: query q is served by GPU q mod G; arrival times kept."""
    return trace[trace["qid"] % world == rank]


def gather_latencies(lat_ms: np.ndarray, world: int, rank: int, dist):
    """All ranks' per-query latencies on rank 0 (C4; None elsewhere)."""
    if world == 1:
        return np.asarray(lat_ms)
    parts = [None] * world
    dist.all_gather_object(parts, np.asarray(lat_ms))
    return np.concatenate(parts) if rank == 0 else None


def p95_nearest_rank(lat_ms: np.ndarray) -> float:
    s = np.sort(np.asarray(lat_ms, dtype=np.float64))
    return float(s[max((95 * s.size + 99) // 100, 1) - 1]) if s.size else float("nan")


def sla_search(model, cfg, world, rank, dist, streams, d, lam0, n, sla_ms, max_iter=10, tau_ms=0.0,
               replicated=False):
    """lambda*: largest offered Poisson rate (all GPUs) with p95 <= SLA and every GPU keeping up
    (S5; geometric bracketing then bisection).  Real clock, device-synth inputs.
    replicated=True (model-parallel sharding): every rank serves the WHOLE trace (the same
    global batches) and the p95 is rank 0's; otherwise replicas serve q mod G."""
    import torch
    probes = []
    count = [0]

    def probe(lam):
        count[0] += 1
        tr = W.poisson_trace(lam, n, seed=12)
        mine = tr if replicated else rank_share(tr, world, rank)
        rep = model.rec_serve(mine, sla_ms, streams, d, fusion_timeout_ms=tau_ms, warmup_frac=0.1)
        lib_global = world > 1 and rep.get("ranks", 1) == world   # the library gathered (C4)
        if not lib_global:
            arr = mine["arrival_s"]
            w_end = tr["arrival_s"][0] + 0.1 * (tr["arrival_s"][-1] - tr["arrival_s"][0])
            mylat = rep["latency_ms"][arr >= w_end]
            lat = mylat if replicated else gather_latencies(mylat, world, rank, dist)
        stable = torch.tensor([rep["stable"]], device="cuda")
        if world > 1:
            dist.all_reduce(stable, op=dist.ReduceOp.MIN)
        ok = torch.tensor([0], device="cuda")
        if rank == 0:
            p95 = rep["p95_ms"] if lib_global else p95_nearest_rank(lat)
            ok[0] = int(stable.item() == 1 and p95 <= sla_ms)
            probes.append({"offered_qps": round(lam), "p95_ms": round(p95, 3), "ok": int(ok.item()),
                           "p95_from": "library (all ranks)" if lib_global else "python gather"})
        if world > 1:
            dist.broadcast(ok, 0)
        return bool(ok.item())

    lo, hi, lam = None, None, lam0
    for _ in range(max_iter):
        if probe(lam):
            lo = lam
            if hi is not None:
                break
            lam *= 2.0
        else:
            hi = lam
            if lo is not None:
                break
            lam *= 0.5
    while lo is not None and hi is not None and (hi - lo) > 0.01 * lo and count[0] < 2 * max_iter:
        mid = 0.5 * (lo + hi)
        if probe(mid):
            lo = mid
        else:
            hi = mid
    return (lo or 0.0), probes


