"""GPU serving tests (a1, a7): rec_serve against the oracle's S1-S5.

* virtual clock: the batch list (stream, qid, start, len per batch) is bit-exact with
  oracle.serving.replay_virtual and latencies equal the oracle's; the CTRs of every
  served item equal a direct rec_query of the same items (batch invariance) and the
  oracle within 2e-2.
* real clock: invariants only (coverage exactly once with S1 boundaries, FIFO,
  sum <= d, conservation, p95 recomputed from the raw per-query latencies).
* host-input mode (PCIe data loading) gives the same CTRs as device-synth.
"""
import numpy as np
import pytest

import workloads as W
from oracle import forward as fw, gen, serving as sv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


CFG = W.small_variant(W.RMC1, 20000)


@pytest.fixture(scope="module")
def model():
    from paper_2203_07424_b200 import RecModel
    m = RecModel(CFG, seed=1, max_batch=256, streams=4)
    yield m
    m.close()


def _batches_from_log(log):
    out = {}
    for b, s, q, st, ln in log:
        out.setdefault(int(b), (int(s), []))[1].append((int(q), int(st), int(ln)))
    return [out[k] for k in sorted(out)]


@pytest.mark.parametrize("streams,d,tau", [(1, 256, 0.0), (3, 128, 0.0), (2, 256, 0.05)])
def test_virtual_clock_bit_exact(model, streams, d, tau):
    tr = W.poisson_trace(4000.0, 150, seed=13)
    alpha, beta = 30000.0, 250.0
    rep = model.rec_serve(tr, 50.0, streams, d, fusion_timeout_ms=tau, clock=1, alpha_ns=alpha,
                          beta_ns=beta, log_cap=100000, want_ctr=True)
    ref = sv.replay_virtual(tr, streams, d, alpha, beta, fusion_timeout_ms=tau)
    got = _batches_from_log(rep["batch_log"])
    exp = [(b["stream"], b["segs"]) for b in ref.batches]
    assert got == exp
    assert np.array_equal(rep["latency_ms"], ref.latency_s * 1e3)
    orep = sv.summarize(tr, ref.latency_s, ref.completion_s, 50.0)
    assert rep["p95_ms"] == orep["p95_ms"] and rep["sla_met"] == orep["sla_met"]
    assert rep["completed"] == len(tr) and rep["batches"] == len(ref.batches)
    # CTRs of served items == oracle (sampled) within 2e-2
    ctr = rep["ctr"]
    base = np.concatenate([[0], np.cumsum(tr["size"].astype(np.int64))])
    rng = np.random.default_rng(1)
    pick_q = rng.choice(len(tr), size=12, replace=False)
    segs = np.array([[tr["qid"][p], 0, tr["size"][p]] for p in pick_q], np.int32)
    ind, off, dense = gen.gen_batch(CFG, 1, segs)
    exp_ctr = fw.forward(CFG, 1, dense, ind, off)
    got_ctr = np.concatenate([ctr[base[p]:base[p + 1]] for p in pick_q])
    assert np.abs(got_ctr - exp_ctr).max() <= 2e-2


def test_real_clock_invariants(model):
    tr = W.poisson_trace(3000.0, 600, seed=14)
    d = 256
    rep = model.rec_serve(tr, 20.0, 4, d, log_cap=100000)
    log = rep["batch_log"]
    assert rep["completed"] == len(tr) and rep["dropped"] == 0
    seen = {}
    for b, s, q, st, ln in log:
        seen.setdefault(int(q), []).append((int(st), int(ln)))
    for p in range(len(tr)):
        assert sorted(seen[int(tr["qid"][p])]) == sv.split(int(tr["size"][p]), d)
    for _, (s, segs) in enumerate(_batches_from_log(log)):
        assert 1 <= sum(x[2] for x in segs) <= d
    order = [(int(q), int(st)) for _, _, q, st, _ in log]
    assert order == sorted(order)                          # FIFO
    lat = rep["latency_ms"]
    assert np.all(lat > 0)
    orep = sv.summarize(tr, lat * 1e-3, tr["arrival_s"] + lat * 1e-3, 20.0)
    assert abs(rep["p95_ms"] - orep["p95_ms"]) < 1e-9
    assert rep["p95_ms"] >= rep["p50_ms"]


def test_host_input_mode_matches_synth(model):
    tr = W.poisson_trace(2000.0, 60, seed=15)
    a = model.rec_serve(tr, 50.0, 2, 256, clock=1, alpha_ns=50000.0, beta_ns=100.0, want_ctr=True)
    b = model.rec_serve(tr, 50.0, 2, 256, clock=1, alpha_ns=50000.0, beta_ns=100.0, want_ctr=True,
                        input_mode=1)
    assert np.array_equal(a["ctr"], b["ctr"])
    assert np.array_equal(a["latency_ms"], b["latency_ms"])


def test_policy_validation(model):
    from paper_2203_07424_b200 import RecError
    tr = W.poisson_trace(1000.0, 10, seed=1)
    for kw in ({"streams": 0, "max_batch": 64}, {"streams": 9, "max_batch": 64},
               {"streams": 1, "max_batch": 0}, {"streams": 1, "max_batch": 100000}):
        with pytest.raises(RecError) as ei:
            model.rec_serve(tr, 20.0, **kw)
        assert ei.value.status == -1


@pytest.mark.parametrize("lanes,nb", [(2, 13), (1, 8)])
def test_pipeline_matches_slots(lanes, nb):
    """S-D pipeline lanes (rec_set_pipeline): the CTRs of every batch are bit-identical to the
    per-stream slot graphs (same kernels, same per-batch buffers), including a remainder
    group that falls back to the slot graphs, and match the oracle on sampled items."""
    import torch
    from paper_2203_07424_b200 import RecModel, rec_split_fuse
    m = RecModel(CFG, seed=1, max_batch=256, streams=4)
    tr = W.burst_trace(60, seed=23)
    segs, bstart = rec_split_fuse(tr, 256)
    bstart = bstart[:nb + 1]
    items = int(segs[:bstart[-1], 2].sum())
    ref = torch.zeros(items, device="cuda")
    off = 0
    for b in range(nb):
        sg = segs[bstart[b]:bstart[b + 1]]
        n = int(sg[:, 2].sum())
        m.rec_synth_query_async(b % 4, sg, ref[off:off + n])
        m.rec_sync(b % 4)
        off += n
    m.rec_set_pipeline(lanes)
    got = torch.full((items,), -1.0, device="cuda")
    for _ in range(2):  # second pass reuses the lane graphs
        m.rec_synth_query_pipeline(segs[:bstart[-1]], bstart, got)
        for k in range(4):
            m.rec_sync(k)
        assert np.array_equal(got.cpu().numpy(), ref.cpu().numpy())
    # back to slot graphs after pipeline mode: same bits
    sg = segs[bstart[0]:bstart[1]]
    n0 = int(sg[:, 2].sum())
    again = torch.zeros(n0, device="cuda")
    m.rec_synth_query_async(1, sg, again)
    m.rec_sync(1)
    assert np.array_equal(again.cpu().numpy(), ref[:n0].cpu().numpy())
    q, it = gen.expand_segments(segs[:bstart[-1]])
    pick = np.random.default_rng(5).choice(items, size=24, replace=False)
    sub = np.array([[q[k], it[k], 1] for k in pick], np.int32)
    i2, o2, d2 = gen.gen_batch(CFG, 1, sub)
    exp = fw.forward(CFG, 1, d2, i2, o2)
    assert np.abs(got.cpu().numpy()[pick] - exp).max() <= 2e-2
    m.close()


def test_pipeline_argument_errors():
    from paper_2203_07424_b200 import RecModel, RecError
    m = RecModel(CFG, seed=1, max_batch=64, streams=3)
    with pytest.raises(RecError):
        m.rec_set_pipeline(2)          # 3 streams do not split into lanes of >= 2
    with pytest.raises(RecError):
        m.rec_synth_query_pipeline(np.array([[0, 0, 4]], np.int32), np.array([0, 1], np.int64))
    m.rec_set_pipeline(0)
    m.close()


def test_concurrent_streams_match_sequential():
    """Co-location: 24 batches submitted back to back over 4 stream slots (device-
    synthesised inputs, and caller host buffers through rec_query_async) give the same CTR
    bits as the same batches run one at a time — no workspace or graph-slot races."""
    import torch
    from paper_2203_07424_b200 import RecModel, rec_split_fuse
    m = RecModel(CFG, seed=1, max_batch=256, streams=4)
    tr = W.burst_trace(200, seed=31)
    segs, bstart = rec_split_fuse(tr, 256)
    nb = min(24, len(bstart) - 1)
    batches = [np.ascontiguousarray(segs[bstart[b]:bstart[b + 1]]) for b in range(nb)]
    n_items = [int(b[:, 2].sum()) for b in batches]
    seq = []
    for b in range(nb):
        c = torch.zeros(n_items[b], device="cuda")
        m.rec_synth_query_async(0, batches[b], c)
        m.rec_sync(0)
        seq.append(c.cpu().numpy())
    outs = [torch.zeros(n, device="cuda") for n in n_items]
    for b in range(nb):                                  # no sync between submissions
        m.rec_synth_query_async(b % 4, batches[b], outs[b])
    for k in range(4):
        m.rec_sync(k)
    for b in range(nb):
        assert np.array_equal(outs[b].cpu().numpy(), seq[b]), b
    # caller inputs from pinned host buffers, 4 streams in flight
    host = [gen.gen_batch(CFG, 1, bt) for bt in batches]
    pins = [[torch.from_numpy(x).pin_memory() for x in h] for h in host]
    res = [torch.zeros(n).pin_memory() for n in n_items]
    for b in range(nb):
        d_, i_, o_ = pins[b][2], pins[b][0], pins[b][1]
        m.rec_query_async(b % 4, d_, i_, o_, int(host[b][1][-1]), n_items[b], res[b])
    for k in range(4):
        m.rec_sync(k)
    for b in range(nb):
        assert np.array_equal(res[b].numpy(), seq[b]), b
    m.close()


def test_mtwnd_serving_ctrs():
    """rec_serve on the MT-WnD model (virtual clock): every served item's N task CTRs equal a
    direct rec_query of the same items (batch invariance) and the oracle within 2e-2."""
    from paper_2203_07424_b200 import RecModel
    cfg = W.small_variant(W.MTWND, 20000)
    m = RecModel(cfg, seed=1, max_batch=128, streams=2)
    tr = W.poisson_trace(2000.0, 40, seed=17)
    rep = m.rec_serve(tr, 100.0, 2, 128, clock=1, alpha_ns=30000.0, beta_ns=250.0, want_ctr=True)
    ctr = rep["ctr"]
    assert rep["completed"] == len(tr) and ctr.shape == (int(tr["size"].sum()), cfg.tasks)
    base = np.concatenate([[0], np.cumsum(tr["size"].astype(np.int64))])
    for q in (0, 7, 21):
        n = int(tr["size"][q])
        take = min(n, 128)
        segs = np.array([[int(tr["qid"][q]), 0, take]], np.int32)
        ind, off, dense = gen.gen_batch(cfg, 1, segs)
        direct = np.zeros((take, cfg.tasks), np.float32)
        m.rec_query(dense, ind, off, take, direct)
        assert np.array_equal(ctr[base[q]:base[q] + take], direct)
        exp = fw.forward(cfg, 1, dense, ind, off)
        assert np.abs(direct - exp).max() <= 2e-2
    m.close()


@pytest.mark.parametrize("mode", ["synth", "host"])
def test_latency_breakdown_components(model, mode):
    """breakdown_ms = (queue, input, sparse, dense), P:418's latency components (recorded while
    profiling is on, rec_profile): every one is
    non-negative, sparse and dense are positive device times, input is positive exactly in the
    host-input (PCIe) mode, and queue + input + sparse + dense stays below the mean latency
    (the rest is launch and completion-observation overhead)."""
    from paper_2203_07424_b200 import REC_INPUT_HOST, REC_INPUT_DEVICE_SYNTH
    tr = W.poisson_trace(3000.0, 300, seed=21)
    im = REC_INPUT_HOST if mode == "host" else REC_INPUT_DEVICE_SYNTH
    model.rec_profile(True)                 # the breakdown is recorded while profiling
    r = model.rec_serve(tr, 1e9, streams=2, max_batch=256, input_mode=im)
    model.rec_profile(False)
    q, inp, sp, de = r["breakdown_ms"]
    assert min(q, inp, sp, de) >= 0
    assert sp > 0 and de > 0
    assert (inp > 0) == (mode == "host")
    assert q + inp + sp + de <= r["mean_ms"] * 1.001 + 1e-6
