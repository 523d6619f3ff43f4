"""a1 host logic (C++ rec_split_fuse, no GPU needed) against the oracle's S1/S2."""
import numpy as np
import pytest

import workloads as W
from oracle import serving as sv


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


def _oracle_batches(trace, d):
    fifo = []
    for r in trace:
        for (s, ln) in sv.split(int(r["size"]), d):
            fifo.append((int(r["qid"]), s, ln))
    out, head = [], 0
    while head < len(fifo):
        k = sv.fuse_head([f[2] for f in fifo[head:head + d + 1]], d)
        out.append(fifo[head:head + k])
        head += k
    return out


@pytest.mark.parametrize("d", [1, 7, 256, 1024])
def test_split_fuse_bit_exact(d):
    from paper_2203_07424_b200 import rec_split_fuse
    tr = W.burst_trace(700, seed=3)
    segs, bs = rec_split_fuse(tr, d)
    got = [[tuple(int(v) for v in segs[i]) for i in range(bs[b], bs[b + 1])] for b in range(len(bs) - 1)]
    assert got == _oracle_batches(tr, d)
    for b in got:
        assert 1 <= sum(s[2] for s in b) <= d


def test_split_fuse_errors():
    from paper_2203_07424_b200 import rec_split_fuse, RecError
    tr = W.burst_trace(5, seed=1)
    with pytest.raises(RecError):
        rec_split_fuse(tr, 0)
    tr["size"][2] = 0
    with pytest.raises(RecError):
        rec_split_fuse(tr, 16)


def test_global_batches_match_oracle_and_invariants():
    """R31 (sharded serving's deterministic dispatcher): the C++ cut equals the oracle's
    step-by-step cut on random Poisson traces (batch lists bit-exact, close times exact), and
    the invariants hold: coverage exactly once with S1 boundaries, FIFO, sum <= d, every batch
    full or closed at first arrival + tau, non-decreasing close times."""
    from paper_2203_07424_b200 import rec_global_batches
    from oracle import serving as sv
    for seed, rate, d, tau in ((1, 2000.0, 1024, 1.0), (2, 30000.0, 256, 0.5), (3, 500.0, 1024, 5.0),
                               (4, 100000.0, 512, 0.2)):
        tr = W.poisson_trace(rate, 400, seed=seed)
        segs, bst, close = rec_global_batches(tr, d, tau)
        osegs, obst, oclose = sv.global_batches(tr["arrival_s"], tr["size"], tr["qid"], d, tau * 1e-3)
        assert np.array_equal(segs, osegs) and np.array_equal(bst, obst)
        assert np.array_equal(close, oclose)
        assert np.all(np.diff(close) >= 0)
        arr = dict(zip(tr["qid"].tolist(), tr["arrival_s"].tolist()))
        for b in range(len(bst) - 1):
            sg = segs[bst[b]:bst[b + 1]]
            items = int(sg[:, 2].sum())
            assert items <= d or len(sg) == 1
            first = arr[int(sg[0, 0])]
            assert close[b] >= first - 1e-15
            if items < d and b + 1 < len(bst) - 1:
                nxt = segs[bst[b + 1]]
                full = items + int(nxt[2]) > d and arr[int(nxt[0])] <= first + tau * 1e-3
                assert full or abs(close[b] - max(first + tau * 1e-3, close[b - 1] if b else -1)) < 1e-12
        # coverage: every query's items exactly once, in S1 chunks
        got = {}
        for q, st, ln in segs:
            got.setdefault(int(q), []).append((int(st), int(ln)))
        for q, n in zip(tr["qid"], tr["size"]):
            assert got[int(q)] == sv.split(int(n), d)
