"""Algorithm 1 of the paper, gradient-based search over the serving policy
space P_sp(M+D) of one GPU: m co-located streams x d max fused batch.

From the origin (least co-location, smallest batch) the search evaluates three
candidates — batch up, streams up, both up — and moves to the one with the largest
latency-bounded-throughput gain while that gain is positive.  `evaluate(m, d)`
returns the SLA-bounded QPS (lambda*) of the policy, which already encodes Alg. 1's latency
constraint (line 665).  Ties prefer fewer streams, then smaller batches.
"""
from typing import Callable, Dict, List, Sequence, Tuple


def _neighbours(i: int, j: int, nm: int, nd: int) -> List[Tuple[int, int]]:
    c = []
    if j + 1 < nd:
        c.append((i, j + 1))          # (1) batch size only
    if i + 1 < nm:
        c.append((i + 1, j))          # (2) co-located streams only
    if i + 1 < nm and j + 1 < nd:
        c.append((i + 1, j + 1))      # (3) both
    return c


def gradient_search(evaluate: Callable[[int, int], float], ms: Sequence[int], ds: Sequence[int],
                    noise: float = 0.0) -> Dict:
    seen: Dict[Tuple[int, int], float] = {}

    def q(p):
        if p not in seen:
            seen[p] = float(evaluate(ms[p[0]], ds[p[1]]))
        return seen[p]

    here = (0, 0)
    trail = [here]
    while True:
        cands = _neighbours(here[0], here[1], len(ms), len(ds))
        if not cands:
            break
        best = cands[0]
        for c in cands[1:]:
            if q(c) > q(best) or (q(c) == q(best) and c < best):
                best = c
        gain = q(best) - q(here)
        if gain > 0 and gain > noise * q(here):
            here = best
            trail.append(here)
        else:
            break
    return {"m": ms[here[0]], "d": ds[here[1]], "qps": q(here), "evals": len(seen),
            "path": [(ms[i], ds[j]) for i, j in trail],
            "evaluated": {f"m{ms[i]}_d{ds[j]}": v for (i, j), v in sorted(seen.items())}}
