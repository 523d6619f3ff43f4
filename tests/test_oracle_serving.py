"""Oracle pins for split / fuse / virtual-clock replay / SLA metric (S1-S5)."""
import numpy as np
import pytest

import workloads as W
from oracle import serving as sv


def _trace(rows):
    tr = np.zeros(len(rows), dtype=W.TRACE_DTYPE)
    for k, (a, s) in enumerate(rows):
        tr[k] = (a, s, k)
    return tr


@pytest.mark.parametrize("n,d", [(1, 1), (5, 1), (1000, 256), (1024, 1024), (1025, 1024), (7, 3)])
def test_split_closed_form(n, d):
    ch = sv.split(n, d)
    k = -(-n // d)
    assert len(ch) == k and sum(c[1] for c in ch) == n
    assert [c[0] for c in ch] == [i * d for i in range(k)]
    assert all(c[1] == d for c in ch[:-1]) and 1 <= ch[-1][1] <= d


def test_fuse_head_cases():
    assert sv.fuse_head([4, 2], 4) == 1
    assert sv.fuse_head([2, 1, 3], 4) == 2
    assert sv.fuse_head([1, 1, 1, 1, 1], 4) == 4
    assert sv.fuse_head([5], 4) == 1        # at least one (cannot happen after split)


def test_p95_nearest_rank_hand_arrays():
    assert sv.p_nearest_rank(np.arange(1, 21), 95) == 19          # ceil(0.95*20) = 19
    assert sv.p_nearest_rank(np.arange(1, 101), 95) == 95
    assert sv.p_nearest_rank([3.0], 95) == 3.0
    assert sv.p_nearest_rank(np.arange(1, 11)[::-1], 50) == 5
    assert sv.p_nearest_rank(np.arange(1, 22), 95) == 20          # ceil(19.95) = 20


def _hand_trace():
    # q0 @0 size 6; q1 @1us size 1; q2 @1us size 3
    return _trace([(0.0, 6), (1e-6, 1), (1e-6, 3)])


def test_replay_hand_traced_one_stream():
    # alpha = 1 us, beta = 0.1 us/item, d = 4, m = 1 (derivation in DESIGN.md §3 S4 example)
    r = sv.replay_virtual(_hand_trace(), 1, 4, 1000.0, 100.0)
    assert [b["segs"] for b in r.batches] == [[(0, 0, 4)], [(0, 4, 2), (1, 0, 1)], [(2, 0, 3)]]
    assert np.allclose(r.latency_s, [2.7e-6, 1.7e-6, 3.0e-6], rtol=1e-12)


def test_replay_hand_traced_two_streams():
    r = sv.replay_virtual(_hand_trace(), 2, 4, 1000.0, 100.0)
    assert [(b["stream"], b["segs"]) for b in r.batches] == [
        (0, [(0, 0, 4)]), (1, [(0, 4, 2)]), (1, [(1, 0, 1), (2, 0, 3)])]
    assert np.allclose(r.latency_s, [1.4e-6, 1.6e-6, 1.6e-6], rtol=1e-12)


def test_replay_fusion_timeout_delays_partial_batch():
    tr = _trace([(0.0, 2)])
    r0 = sv.replay_virtual(tr, 1, 4, 1000.0, 100.0, fusion_timeout_ms=0.0)
    r1 = sv.replay_virtual(tr, 1, 4, 1000.0, 100.0, fusion_timeout_ms=1e-3)   # tau = 1 us
    assert np.isclose(r0.latency_s[0], 1.2e-6) and np.isclose(r1.latency_s[0], 2.2e-6)
    # a full batch fires immediately even with a timeout
    r2 = sv.replay_virtual(_trace([(0.0, 4)]), 1, 4, 1000.0, 100.0, fusion_timeout_ms=1.0)
    assert np.isclose(r2.latency_s[0], 1.4e-6)


def test_replay_invariants_random_trace():
    tr = W.poisson_trace(20000.0, 600, seed=11)
    d = 256
    r = sv.replay_virtual(tr, 3, d, 20000.0, 15.0)
    # coverage exactly once with S1 boundaries; FIFO order; sum <= d
    seen = {}
    order = []
    for b in r.batches:
        assert 1 <= sum(s[2] for s in b["segs"]) <= d
        for (q, s, ln) in b["segs"]:
            seen.setdefault(q, []).append((s, ln))
            order.append((q, s))
    for q in range(len(tr)):
        assert sorted(seen[q]) == sv.split(int(tr["size"][q]), d)
    assert order == sorted(order, key=lambda x: (x[0], x[1]))      # FIFO = qid then start
    assert np.all(np.isfinite(r.latency_s)) and np.all(r.latency_s > 0)
    # each query's latency >= its service lower bound
    assert np.all(r.latency_s >= (20000.0 + 15.0) * 1e-9 - 1e-15)


def test_rate_to_zero_gives_service_time():
    # arrival rate -> 0 => tail latency -> single-query service time
    tr = _trace([(k * 1.0, 100) for k in range(50)])
    r = sv.replay_virtual(tr, 1, 1024, 5000.0, 10.0)
    assert np.allclose(r.latency_s, (5000.0 + 10.0 * 100) * 1e-9, rtol=1e-9)


def test_lambda_star_bracketing_bisection():
    thr = 123456.0
    lam = sv.lambda_star(lambda x: x <= thr, 1000.0)
    assert thr * 0.99 <= lam <= thr
    lam = sv.lambda_star(lambda x: x <= thr, 1e7)
    assert thr * 0.99 <= lam <= thr
    # SLA below single-query service time => lambda* = 0
    assert sv.lambda_star(lambda x: False, 1000.0) == 0.0


def _probe_factory(sla_ms, alpha_ns, beta_ns, m=2, d=256, n=800, seed=3):
    def probe(lam):
        tr = W.poisson_trace(lam, n, seed)
        r = sv.replay_virtual(tr, m, d, alpha_ns, beta_ns)
        rep = sv.summarize(tr, r.latency_s, r.completion_s, sla_ms)
        return rep["sla_met"] == 1
    return probe


def test_sla_infinite_is_saturation_and_tiny_sla_is_zero():
    # SLA = inf => lambda* is limited only by saturation: it exceeds any finite-SLA lambda*
    a, b = 20000.0, 20.0
    lam_inf = sv.lambda_star(_probe_factory(1e12, a, b), 1000.0, lam_min=1.0)
    lam_fin = sv.lambda_star(_probe_factory(0.2, a, b), 1000.0, lam_min=1.0)
    assert lam_inf >= lam_fin > 0
    # SLA below the single-query service time (alpha alone = 20 us) => 0
    assert sv.lambda_star(_probe_factory(0.01, a, b), 1000.0, lam_min=1.0) == 0.0


def test_summarize_tail_ge_mean_and_achieved_le_offered():
    tr = W.poisson_trace(5000.0, 500, seed=2)
    r = sv.replay_virtual(tr, 2, 512, 30000.0, 10.0)
    rep = sv.summarize(tr, r.latency_s, r.completion_s, 50.0)
    assert rep["p95_ms"] >= rep["p50_ms"] and rep["p99_ms"] >= rep["p95_ms"]
    assert rep["achieved_qps"] <= rep["offered_qps"] * 1.0001 + 1e-9
    assert rep["completed"] == 500
