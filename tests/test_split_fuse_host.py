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
