"""bench.py — throughput of the B200 DLRM query hot path (Hercules, arXiv 2203.07424).

One JSON line on rank 0.  Workload (N = 1): BASELINE.json configs[1], DLRM-RMC1 —
10 tables x 1M rows x dim 32 (1.28 GB fp32, >> 126 MB L2), pooling 80, bottom
256-128-32, top 256-64-1, fused batches of d = 1024 items on 16 co-located streams.

A STEP = one serving round of --step-batches (512) fused batches: a1 (queries of a burst
trace, split/fused into batches of <= d by the library's C++ splitter/fuser before timing),
then per batch a2 (device-side generation of its indices and dense features from (seed,
qid, item)), a3 SLS, a4 bottom MLP, a5 dot interaction, a6 top MLP + sigmoid, the batches
dealt round-robin to the co-located streams.  `value` = queries completed per
second (a query completes when its last sub-query's batch is done) = whole-job throughput
summed over ranks (replicas, no data-path collective: scaling "weak").  It is the saturation
(SLA-unbounded) QPS; the serving run that checks the p95 SLA (Alg. 1 over streams x d) is
`sla`, and `per_model` repeats saturation / SLS roofline / lambda* for RMC2, RMC3, MT-WnD.

`e2e` is the same metric through rec_query_async with HOST buffers (indices, offsets, dense
copied host->device and the CTRs device->host for every batch).  `roofline` is the SLS kernel:
algorithmic bytes / its CUDA-event time on its own stream (plus the in-step
aggregate and the caller-index kernel).  `cpu_baseline` times the CPU oracle on the host cores
on a bounded sample.  `--gpus N` re-executes under torch.distributed.run; `--shard table`
measures table-wise sharded serving instead of replicas.

--impl reference runs the CPU oracle (the tier's reference arm) as the timed program.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# hardware work queues shared by the co-located streams (must precede CUDA initialisation;
# measured RMC1 flat, RMC3 +1.7 % at 32 vs the default 8: scripts/ab_conn.sh)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import workloads as W  # noqa: E402

BASELINE_METRIC = "SLA-bounded QPS (p95) per model at 1/2/4/8 B200; SLS HBM GB/s; MLP TC util"
# saturation_ge_lambda_star: saturation >= LAMBDA_TOL x lambda*.  lambda* is resolved to 2 %
# by the bisection and a finite Poisson trace passes as "stable" when it achieves >= 98 % of
# the offered rate (csrc/serve.cpp), so a passing probe can sit up to ~4 % above the
# steady-state capacity the saturation step measures.
LAMBDA_TOL = 0.96


def sls_bytes_per_item(cfg, synth: bool = False) -> int:
    """Algorithmic bytes of the SLS per item: T*L fp32 rows of D + int32 indices
    + int32 offsets + the fp32 pooled write.  synth=True: the serving/bench kernel generates
    its indices in-kernel (fixed pooling), so no index / offset array is read."""
    T, L, D = cfg.num_tables, 0.5 * (cfg.pooling_lo + cfg.pooling_hi), cfg.dim
    if synth and cfg.pooling_lo == cfg.pooling_hi:
        return int(T * L * D * 4 + T * D * 4)
    return int(T * (L * D * 4 + L * 4 + 4) + T * D * 4)


def mlp_flops_per_item(cfg) -> int:
    """2 * sum(fan_in * fan_out) over the bottom MLP and every top stack / task tower (+ the
    MT-WnD wide dot products)."""
    f = 0
    for a, b in zip(cfg.bottom[:-1], cfg.bottom[1:]):
        f += 2 * a * b
    widths = [cfg.top_in] + list(cfg.top)
    tower = sum(2 * a * b for a, b in zip(widths[:-1], widths[1:]))
    wide = 2 * cfg.top_in if cfg.arch == W.ARCH_MTWND else 0
    return f + cfg.tasks * (tower + wide)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d.get("bf16_tflops"), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region, in-process through NVML
    (a background thread polling every 10 ms; nvidia-smi's own -lms loop as a fallback when
    NVML is unavailable).  mark(t0, t1) brackets the timed region."""

    HW, HWT, SWT, SWP = 0x8, 0x40, 0x20, 0x4   # nvmlClocksEventReason* bits

    def __init__(self, dev: int, period_s: float = 0.01):
        self.dev, self.period, self.samples, self.proc = dev, period_s, [], None
        self._stop = threading.Event()
        self.backend = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.dev)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            get_r = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def loop():
                while not self._stop.is_set():
                    try:
                        self.samples.append((time.perf_counter(),
                                             float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                                             int(get_r(h))))
                    except Exception:
                        pass
                    self._stop.wait(self.period)
            self.backend = "nvml"
        except Exception:
            self.max_mhz = None
            q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
            try:
                self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}",
                                              "--format=csv,noheader,nounits", "-lms", "20"],
                                             stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except FileNotFoundError:
                return self

            def loop():
                for line in self.proc.stdout:
                    f = [x.strip() for x in line.split(",")]
                    try:
                        self.max_mhz = float(f[1])
                        self.samples.append((time.perf_counter(), float(f[0]), int(f[2], 16)))
                    except (ValueError, IndexError):
                        pass
            self.backend = "nvidia-smi"
        self.t = threading.Thread(target=loop, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        """Median SM clock + throttle reasons of the samples inside [t0, t1]; when the region
        is shorter than the sampling period, the samples of the whole load window."""
        inside = [x for x in self.samples if t0 is not None and t0 <= x[0] <= t1]
        rows = inside or list(self.samples)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0,
                    "backend": self.backend}
        names = {self.HW: "hw_slowdown", self.HWT: "hw_thermal_slowdown",
                 self.SWT: "sw_thermal_slowdown", self.SWP: "sw_power_cap"}
        reasons = sorted({n for _, _, r in rows for bit, n in names.items() if r & bit})
        return {"sm_mhz": statistics.median(x[1] for x in rows), "sm_max_mhz": self.max_mhz,
                "sm_mhz_min": min(x[1] for x in rows), "reasons": reasons, "samples": len(rows),
                "window": "timed region" if inside else "load window", "backend": self.backend}


# ------------------------------------------------------------------ CPU oracle timing
def _oracle_forward_job(args):
    """One oracle forward (fp64, oracle/forward.py) over pre-generated inputs; returns its own
    CPU time and item count.  Input generation is NOT timed (it happens in the parent before
    the timed region, as the GPU arm's inputs are resident when its timed region starts)."""
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    name, ind, off, dense, seed = args
    from oracle import forward
    cfg = W.SHORT[name]
    t = time.perf_counter()
    forward.forward(cfg, seed, dense, ind, off)
    return time.perf_counter() - t, int(dense.shape[0])


def _oracle_inputs(name: str, items: int, seed: int):
    from oracle import gen
    cfg = W.SHORT[name]
    ind, off, dense = gen.gen_batch(cfg, 1, W.random_segments(items, seed=seed))
    return (name, ind, off, dense, 1)


def _pool(cores: int):
    import multiprocessing as mp
    os.environ["OMP_NUM_THREADS"] = "1"          # inherited by the forked workers
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    return mp.get_context("fork").Pool(cores)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_baseline(name: str, items_per_job: int, jobs_per_core: int, cores: int) -> dict:
    """cpu_baseline: the oracle as it stands on a warm process pool (one process per core),
    inputs generated before the timed map; items/s = items / wall of the timed map.  The
    1-core figure is items / the summed per-job forward times."""
    work = [_oracle_inputs(name, items_per_job, 100 + j) for j in range(cores * jobs_per_core)]
    with _pool(cores) as pool:
        pool.map(_oracle_forward_job, work[:cores])          # warm the workers (imports, BLAS)
        t0 = time.perf_counter()
        res = pool.map(_oracle_forward_job, work)
        wall = time.perf_counter() - t0
    items = sum(r[1] for r in res)
    return {"items_per_s": items / wall, "items_per_s_1core": items / sum(r[0] for r in res),
            "wall_s": wall, "cpu_s": sum(r[0] for r in res), "items": items}


# largest max-batch d the serving search may pick (BASELINE configs[1]: RMC1 batch 256-1024)
SEARCH_D_MAX = {"DLRM-RMC1": 1024, "DLRM-tiny": 64}

from harness.sla import rank_share, gather_latencies, p95_nearest_rank, sla_search  # noqa: E402
from harness.schedsearch import gradient_search  # noqa: E402


# ---------------------------------------------------------------------- reference arm
def run_reference(args):
    """The tier's reference arm: the CPU oracle (fp64 forward) as it stands, on the host cores,
    one process per core (warm fork pool).  Each step = one job per core of ipj items; inputs
    of every step are generated before the timed region (the GPU arm's inputs are resident in
    HBM when its timed region starts).  ipj is sized from the warm-up so the K timed steps take
    about --ref-budget-s seconds."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = W.SHORT[args.config]
    cores = host_cores()
    mean_q = float(W.query_sizes(200000, seed=11).mean())
    ipj = max(1, args.ref_items // cores)
    with _pool(cores) as pool:
        warm = [_oracle_inputs(args.config, ipj, 7000 + j) for j in range(cores)]
        t0 = time.perf_counter()
        for _ in range(max(args.warmup, 1)):
            pool.map(_oracle_forward_job, warm)
        t_step = (time.perf_counter() - t0) / max(args.warmup, 1)
        if args.steps * t_step > args.ref_budget_s:   # shrink the per-step sample to fit
            ipj = max(1, int(ipj * args.ref_budget_s / (args.steps * t_step)))
        elif args.steps * t_step < 0.25 * args.ref_budget_s:  # grow it (amortise pool overhead)
            ipj = int(ipj * min(16.0, 0.25 * args.ref_budget_s / max(args.steps * t_step, 1e-3)))
        steps_in = [[_oracle_inputs(args.config, ipj, 1000 * (k + 1) + j) for j in range(cores)]
                    for k in range(args.steps)]
        t0 = time.perf_counter()
        items = cpu_s = 0
        for k in range(args.steps):
            for dt, n in pool.map(_oracle_forward_job, steps_in[k]):
                items += n
                cpu_s += dt
        wall = time.perf_counter() - t0
    ips = items / wall
    qps = ips / mean_q
    line = {"impl": "reference", "metric": BASELINE_METRIC, "value": qps, "unit": "QPS",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * wall / max(args.steps, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "items_per_step": items // max(args.steps, 1),
                       "mean_query_items": mean_q, "items_per_s": ips},
            "cpu_baseline": {"value": qps, "unit": "QPS", "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "value_1core": (items / cpu_s) / mean_q if cpu_s > 0 else None,
                             "sample": f"{items // max(args.steps, 1)} items/step of {cfg.name} "
                                       f"({cores} jobs x {ipj} items), oracle fp64 forward "
                                       f"(SLS+MLP+interaction+sigmoid) in a warm {cores}-process "
                                       f"pool, inputs generated before the timed region"},
            "e2e": {"value": qps, "unit": "QPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------- our arm
def saturation(model, cfg, d, m_streams, steps, warmup, step_batches, n_queries, rank, world, dist,
               submit="batch", pipe=0, clk=None, sharded=False):
    """Saturation throughput of one replica model (the bench's `value`).

    a1: a burst trace (all queries pending) is split into sub-queries of <= d items and fused
    FIFO into batches of <= d by the library's C++ splitter/fuser (before timing).  A STEP is
    one serving round of `step_batches` fused batches dealt round-robin to the m co-located
    streams, each batch running a2-a6 as one captured graph.  Warm-up runs
    `warmup` such rounds; the timed region (barrier + synchronize on both sides, CUDA events
    on the streams, max over ranks) runs exactly `steps` rounds back to back.  A step of many
    batches keeps the streams loaded so the timed region measures the steady state, not the
    ramp of an idle GPU.  sharded=True: every rank runs the SAME global
    batches (model-parallel embeddings), so items / queries are counted once, not summed."""
    import torch
    from paper_2203_07424_b200 import rec_split_fuse
    dev = torch.device("cuda", torch.cuda.current_device())
    streams = [torch.cuda.ExternalStream(model.rec_stream_handle(k), device=dev) for k in range(m_streams)]
    stream = streams[0]
    trace = W.burst_trace(n_queries, seed=11 + (0 if sharded else rank))
    segs, bstart = rec_split_fuse(trace, d)
    nb = len(bstart) - 1
    sizes = trace["size"].astype(np.int64)
    last_chunk_start = ((sizes - 1) // d) * d
    batches, items_b, done_b = [], [], []
    for b in range(nb):
        sg = segs[bstart[b]:bstart[b + 1]]
        batches.append(np.ascontiguousarray(sg))
        items_b.append(int(sg[:, 2].sum()))
        done_b.append(int(np.sum(sg[:, 1] == last_chunk_start[sg[:, 0]])))

    def sync_all():
        for k in range(m_streams):
            model.rec_sync(k)

    w0, nbt = warmup * step_batches, steps * step_batches
    wl = [batches[i % nb] for i in range(0, w0)]
    tl = [batches[i % nb] for i in range(w0, w0 + nbt)]
    cat = lambda L: (np.concatenate(L).astype(np.int32),
                     np.concatenate([[0], np.cumsum([len(x) for x in L])]).astype(np.int64))
    wsegs, wbstart = cat(wl)
    tsegs, tbstart = cat(tl)
    model.rec_synth_query_batches(wsegs, wbstart, first_slot=0)      # warm-up rounds
    sync_all()
    if pipe > 0:
        model.rec_set_pipeline(pipe)
        model.rec_synth_query_batches(wsegs, wbstart)                # warm the lane graphs
        sync_all()
    base_launch = model.rec_profile_read(4)[1]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    t_region0 = time.perf_counter()
    ev0.record(stream)
    for s in streams[1:]:
        s.wait_event(ev0)                    # fork: every stream starts after ev0
    t_host0 = time.perf_counter()
    if submit == "batch":
        # the library's C++ dispatch loop: one call submits all timed batches round-robin
        model.rec_synth_query_batches(tsegs, tbstart, first_slot=w0 % m_streams)
    else:
        for i in range(w0, w0 + nbt):
            model.rec_synth_query_async(i % m_streams, batches[i % nb], None)
    host_submit_s = time.perf_counter() - t_host0
    for s in streams[1:]:
        e = torch.cuda.Event()
        e.record(s)
        stream.wait_event(e)                 # join: ev1 after every stream's last batch
    ev1.record(stream)
    sync_all()
    torch.cuda.synchronize()
    t_region1 = time.perf_counter()
    if world > 1:
        dist.barrier()
    if pipe > 0:
        model.rec_set_pipeline(0)
    ms = ev0.elapsed_time(ev1)
    launches = model.rec_profile_read(4)[1] - base_launch
    idx = [i % nb for i in range(w0, w0 + nbt)]
    t = torch.tensor([ms, sum(items_b[i] for i in idx), sum(done_b[i] for i in idx)],
                     dtype=torch.float64, device="cuda")
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        if not sharded:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        ms_max = float(tmax[0])
    else:
        ms_max = ms
    return {"ms_max": ms_max, "items": float(t[1]), "queries": float(t[2]), "launches": int(launches),
            "host_submit_s": host_submit_s, "t0": t_region0, "t1": t_region1, "batches": batches,
            "nb": nb, "items_b": items_b, "done_b": done_b, "sizes": sizes, "tsegs": tsegs, "tbstart": tbstart,
            "timed_batches": nbt, "value": float(t[2]) / (ms_max * 1e-3)}


def mlp_large_batch(cfg, mb: int, local: int):
    """MLP utilisation at a large batch (north_star "MLP at >= 60 % of bf16 tensor-pipe peak"):
    the model's bottom and top stacks in a handle with max_batch = mb (tiny tables: the SLS is
    not involved), 20 back-to-back launches of each stage (CUDA events).  Each stack is judged
    against the roofline that binds it: its algorithmic flops / its minimal HBM bytes (bf16
    input row read, output written: the fp32 X slot of the bottom, the CTR of the top) against
    the ridge point bf16 peak / HBM peak; RMC1's narrow stacks are memory-bound, RMC3's
    2560-wide bottom is compute-bound."""
    from paper_2203_07424_b200 import RecModel
    hbm, bf16, _ = peaks()
    mm = RecModel(cfg.with_(rows=1000), seed=1, max_batch=mb, streams=1, device=local)
    fb = sum(2 * x * y for x, y in zip(cfg.bottom[:-1], cfg.bottom[1:]))
    wt = [cfg.top_in] + list(cfg.top)
    ft = cfg.tasks * sum(2 * x * y for x, y in zip(wt[:-1], wt[1:]))
    tb = mm.rec_bench_mlp(0, mb, 20) if fb else 0.0
    ti = mm.rec_bench_mlp(2, mb, 20)
    tt = mm.rec_bench_mlp(1, mb, 20)
    mm.close()

    def judge(flops, nbytes, ms):
        tf = flops * mb / (ms * 1e-3) / 1e12
        gbs = nbytes * mb / (ms * 1e-3) / 1e9
        bound = "tensor" if flops / nbytes > bf16 * 1e3 / hbm else "hbm"
        frac = tf / bf16 if bound == "tensor" else gbs / hbm
        return {"us": 1e3 * ms, "tflops": tf, "tensor_frac": tf / bf16, "gbs": gbs, "bound": bound,
                "frac": frac, "flops_per_item": flops, "min_bytes_per_item": nbytes}
    return {"batch": mb,
            "bottom": judge(fb, 2 * cfg.bottom[0] + 4 * cfg.dim, tb) if fb else None,
            "top": judge(ft, 2 * cfg.top_in + 4 * cfg.tasks, tt - ti),
            "measured": "rec_bench_mlp: 20 back-to-back launches of each stage on one stream (CUDA "
                        "events); top = (interaction + top) - interaction"}


def default_streams(args, name: str) -> int:
    """Co-located streams m for the saturation step: --streams, or per workload
    (profiles/r02/ab_*.txt: RMC3 16 -> 32 streams +16 %; RMC1 flat from 16; RMC2 replicas
    4 / 8 / 16: 30.0k / 29.9k / 29.0k QPS - its 1.23 MB-per-item gathers lose DRAM efficiency
    with more concurrent batches - so 8; sharded RMC2 keeps 16 exchange slots)."""
    if not getattr(args, "streams_auto", False) and args.streams > 0:
        return args.streams
    if name == "rmc2" and getattr(args, "shard", "replica") == "replica":
        return 8
    return 32 if name == "rmc3" else 16


def per_model(name, args, rank, world, dist, local, hbm_peak):
    """The metric is per model (BASELINE.json: "SLA-bounded QPS (p95) per model at 1/2/4/8
    B200"): saturation QPS (the same step definition at fewer steps), the SLS roofline of
    back-to-back launches, and lambda* at the model's paper SLA for the saturation
    step's co-location (m = 16; RMC2 8, RMC3 32) and d = 1024 (the Alg. 1 search runs for the headline
    model)."""
    import torch
    from paper_2203_07424_b200 import RecModel
    cfg = W.SHORT[name]
    d, m_streams = 1024, default_streams(args, name)
    model = RecModel(cfg, seed=1, max_batch=d, streams=m_streams, device=local)
    clk = ClockSampler(local).__enter__()
    sat = saturation(model, cfg, d, m_streams, args.pm_steps, 2, args.pm_step_batches,
                     args.queries, rank, world, dist)
    clk.__exit__(None, None, None)
    out = {"workload": cfg.name, "value": sat["value"], "unit": "QPS", "steps": args.pm_steps,
           "step_batches": args.pm_step_batches, "ms_per_step": sat["ms_max"] / args.pm_steps,
           "items_per_s": sat["items"] / (sat["ms_max"] * 1e-3), "max_batch_d": d,
           "streams": m_streams, "clocks": clk.summary(sat["t0"], sat["t1"])}
    nb = min(sat["timed_batches"], 200)
    if cfg.pooling_fixed:
        tsegs, tbstart = sat["tsegs"], sat["tbstart"]
        bseg = tsegs[:tbstart[nb]]
        b_ms = model.rec_bench_sls(bseg, tbstart[:nb + 1], pdl=True)
        gbs = sls_bytes_per_item(cfg, synth=True) * int(bseg[:, 2].sum()) / (b_ms * 1e-3) / 1e9
        out["sls_roofline"] = {"kernel": "k_sls_synth", "achieved": gbs, "peak": hbm_peak,
                               "unit": "GB/s", "frac": gbs / hbm_peak, "launches": nb,
                               "measured": "rec_bench_sls, PDL back to back, CUDA events"}
    out["sls_in_step_frac"] = (sls_bytes_per_item(cfg, synth=True) * sat["items"] /
                               (sat["ms_max"] * 1e-3) / 1e9 / world / hbm_peak)
    out["mlp_in_step_frac"] = (mlp_flops_per_item(cfg) * sat["items"] / (sat["ms_max"] * 1e-3) /
                               1e12 / world / peaks()[1])
    if args.pm_sla:
        n = int(max(30000, 1.5 * sat["value"]))
        ms = min(m_streams, 16 if name != "rmc3" else 32)   # the saturation step's co-location
        lam, pr = sla_search(model, cfg, world, rank, dist, ms, d, 0.5 * sat["value"], n, cfg.sla_ms)
        out["sla"] = {"sla_ms": cfg.sla_ms, "lambda_star_qps": lam, "policy": {"streams": ms, "max_batch": d},
                      "queries_per_probe": n, "probes": pr,
                      "saturation_ge_lambda_star": bool(sat["value"] >= LAMBDA_TOL * lam)}
    model.close()
    torch.cuda.synchronize()
    if args.mlp_batch > 0 and rank == 0 and name == "rmc3":
        out["mlp_large_batch"] = mlp_large_batch(cfg, args.mlp_batch, local)
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2203_07424_b200 import RecModel, rec_split_fuse, KERNEL_SLS, KERNEL_GEMM

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = W.SHORT[args.config]
    d = args.batch
    m_streams = default_streams(args, args.config)
    l2p = int(args.l2_persist_mb) << 20
    nid = None
    if world > 1:  # replicas: a communicator only for rec_serve's all-rank percentiles (C4)
        from paper_2203_07424_b200 import nccl_unique_id
        t = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(t, 0)
        nid = bytes(t.cpu().numpy())
    model = RecModel(cfg, seed=1, max_batch=d, streams=m_streams, device=local, l2_persist_bytes=l2p,
                     rank=rank, world=world, nccl_id=nid)
    dev = torch.device("cuda", local)
    streams = [torch.cuda.ExternalStream(model.rec_stream_handle(k), device=dev) for k in range(m_streams)]
    stream = streams[0]

    clk = ClockSampler(local).__enter__()
    sat = saturation(model, cfg, d, m_streams, args.steps, args.warmup, args.step_batches,
                     args.queries, rank, world, dist, submit=args.submit, pipe=args.pipe)
    batches, nb, items_b, sizes = sat["batches"], sat["nb"], sat["items_b"], sat["sizes"]
    done_b = sat["done_b"]
    tsegs, tbstart, nbt = sat["tsegs"], sat["tbstart"], sat["timed_batches"]
    ms_max, tot_items, tot_q = sat["ms_max"], sat["items"], sat["queries"]
    launches, host_submit_s = sat["launches"], sat["host_submit_s"]
    t_region0, t_region1 = sat["t0"], sat["t1"]
    w0 = args.warmup * args.step_batches        # first timed batch

    def step(i, slot=None):
        model.rec_synth_query_async(i % m_streams if slot is None else slot, batches[i % nb], None)

    def sync_all():
        for k in range(m_streams):
            model.rec_sync(k)

    # roofline pass: the first timed batches on ONE stream with per-stage CUDA events recorded
    # on that stream around every kernel class (SLS alone on the GPU -> per-launch duration)
    rsteps = min(nbt, args.roofline_steps)
    model.rec_profile(True)
    for i in range(w0, w0 + rsteps):
        step(i, slot=0)
    sls_ms, sls_n = model.rec_profile_read(KERNEL_SLS)
    gemm_ms, gemm_n = model.rec_profile_read(KERNEL_GEMM)
    int_ms, _ = model.rec_profile_read(2)
    gen_ms, _ = model.rec_profile_read(3)
    # back-to-back launch pass: the SLS kernel alone, one launch per batch of the timed
    # sequence (CUDA events on its stream; with and without PDL between launches)
    model.rec_profile(False)
    b2b_n = min(nbt, args.sls_batches)
    bseg = tsegs[:tbstart[b2b_n]]
    b2b_ms = model.rec_bench_sls(bseg, tbstart[:b2b_n + 1], pdl=True)
    ser_ms = model.rec_bench_sls(bseg, tbstart[:b2b_n + 1], pdl=False)
    b2b_bytes = float(sls_bytes_per_item(cfg, synth=True) * int(bseg[:, 2].sum()))
    # caller-index SLS (k_sls: device-resident indices + offsets, the rec_query / e2e path):
    # back-to-back plain launches over distinct full batches of d items
    caller = None
    if args.caller_batches > 0:
        nbc = args.caller_batches
        gi, go = [], []
        for k in range(nbc):
            ind, off, _ = model.rec_gen_batch(np.array([[900000 + k, 0, d]], np.int32))
            gi.append(ind)
            go.append(off)
        stride = max(x.size for x in gi)
        idx_all = np.zeros((nbc, stride), np.int32)
        for k, x in enumerate(gi):
            idx_all[k, :x.size] = x
        di = torch.from_numpy(idx_all).cuda()
        do = torch.from_numpy(np.stack(go)).cuda()
        c_ms = model.rec_bench_sls_caller(di, do, d, nbc, stride)
        c_bytes = sls_bytes_per_item(cfg, synth=False) * d * nbc
        c_gbs = c_bytes / (c_ms * 1e-3) / 1e9
        caller = {"kernel": "k_sls (caller indices)", "achieved": c_gbs, "unit": "GB/s",
                  "frac": c_gbs / peaks()[0], "bytes_per_item": sls_bytes_per_item(cfg, synth=False),
                  "avg_launch_us": 1e3 * c_ms / nbc, "launches": nbc, "batch": d,
                  "measured": "rec_bench_sls_caller: distinct device-resident batches, plain launches "
                              "back to back, CUDA events on the launching stream"}
        del di, do

    # host cost of the submit path (all streams, C++ loop, production graphs)
    hsteps = min(nbt, 1000)
    hb = tbstart[:hsteps + 1]
    model.rec_profile(True)
    model.rec_synth_query_batches(tsegs[:hb[-1]], hb, first_slot=0)
    sync_all()
    host_prof = {k: 1e3 * model.rec_profile_read(5 + j)[0] / hsteps
                 for j, k in enumerate(["param_update_us", "graph_launch_us", "slot_wait_us", "total_us"])}
    model.rec_profile(False)
    clk.__exit__(None, None, None)
    ridx = [i % nb for i in range(w0, w0 + rsteps)]
    ritems = sum(items_b[i] for i in ridx)
    value = tot_q / (ms_max * 1e-3)

    hbm_peak, bf16_peak, peak_kind = peaks()
    traffic = None  # ncu dram__bytes_read.sum + dram__bytes_write.sum per SLS launch (committed capture)
    tp = os.path.join(ROOT, "profiles", "sls_traffic.json")
    tj = json.load(open(tp)) if os.path.exists(tp) else {}
    tj = tj.get("by_workload", {}).get(cfg.name, tj if cfg.name in tj.get("workload", "") else {})
    if tj:
        per_item = tj.get("dram_bytes_per_item")
        if per_item:  # scaled to the mean batch of the measured launches
            traffic = per_item * (b2b_bytes / sls_bytes_per_item(cfg, synth=True)) / max(b2b_n, 1)
    sls_bytes = sls_bytes_per_item(cfg, synth=True) * ritems
    sls_gbs_isolated = sls_bytes / (sls_ms * 1e-3) / 1e9 if sls_ms > 0 else None
    sls_gbs = b2b_bytes / (b2b_ms * 1e-3) / 1e9 if b2b_ms > 0 else None
    sls_gbs_ser = b2b_bytes / (ser_ms * 1e-3) / 1e9 if ser_ms > 0 else None
    flops = mlp_flops_per_item(cfg) * ritems
    gemm_tf = flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None

    # e2e: the same metric through the public query API with HOST buffers: every step copies
    # its inputs (indices, offsets, dense; pinned host memory) to the device and its CTRs
    # back, on the co-located streams (rec_query_async with host pointers, rec_sync at the end)
    e2e = None
    if args.e2e_steps > 0:
        host = []
        for b in range(min(nb, 32)):
            ind, off, dense = model.rec_gen_batch(batches[b])
            host.append((torch.from_numpy(dense).pin_memory(), torch.from_numpy(ind).pin_memory(),
                         torch.from_numpy(off).pin_memory(), int(off[-1]), items_b[b], done_b[b]))
        outs = [torch.empty(d * cfg.tasks, dtype=torch.float32).pin_memory() for _ in range(m_streams)]
        for i in range(2 * m_streams):
            h = host[i % len(host)]
            model.rec_query_async(i % m_streams, h[0], h[1], h[2], h[3], h[4], outs[i % m_streams])
        sync_all()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        q_e2e, h2d, d2h = 0, 0, 0
        nb_e2e = args.e2e_steps * args.step_batches   # steps of step_batches batches, as above
        for i in range(nb_e2e):
            h = host[i % len(host)]
            model.rec_query_async(i % m_streams, h[0], h[1], h[2], h[3], h[4], outs[i % m_streams])
            q_e2e += h[5]
            h2d += h[0].numel() * 4 + h[1].numel() * 4 + h[2].numel() * 4
            d2h += 4 * h[4] * cfg.tasks
        sync_all()
        wall = time.perf_counter() - t0
        tw = torch.tensor([wall, q_e2e], dtype=torch.float64, device="cuda")
        if world > 1:
            twm = tw.clone()
            dist.all_reduce(twm, op=dist.ReduceOp.MAX)
            dist.all_reduce(tw, op=dist.ReduceOp.SUM)
            wall = float(twm[0])
        e2e = {"value": float(tw[1]) / wall, "unit": "QPS",
               "h2d_bytes_per_step": int(h2d / args.e2e_steps),
               "d2h_bytes_per_step": int(d2h / args.e2e_steps),
               "steps": args.e2e_steps, "batches_per_step": args.step_batches,
               "api": f"rec_query_async with pinned host inputs/outputs on {m_streams} streams "
                      f"(H2D of indices/offsets/dense + D2H of CTRs of every batch), wall clock, "
                      f"max over ranks; a step = {args.step_batches} fused batches as in `value`"}

    sla = None
    if args.sla_queries > 0:
        # Alg. 1 over the serving policy (m streams x d max batch); each point is
        # evaluated by its SLA-bounded QPS lambda* (real-clock rec_serve, p95 <= SLA)
        probes_all = {}
        lam_hint = [0.5 * value]

        def evaluate(m, dd):
            lam, pr = sla_search(serve_model, cfg, world, rank, dist, m, dd, lam_hint[0],
                                 args.sla_queries * world, cfg.sla_ms, tau_ms=args.fusion_timeout_ms)
            probes_all[f"m{m}_d{dd}"] = pr
            if lam > 0:
                lam_hint[0] = lam
            return lam

        ms = [x for x in (1, 2, 4, 8, 16, 32) if x <= m_streams]
        # the policy's maximum fusion batch d ("maximum batch sizes fusing queries",
        # bounded only by the SLA); RMC1's BASELINE config fixes 256-1024 (reading R30)
        d_max = args.max_batch_search or SEARCH_D_MAX.get(cfg.name, 4096)
        ds = [x for x in (256, 512, 1024, 2048, 4096) if x <= max(d, d_max)]
        serve_model = model
        if max(ds) > d:  # a second handle with the larger workspaces (tables are regenerated)
            nid2 = None
            if world > 1:
                from paper_2203_07424_b200 import nccl_unique_id
                t2 = torch.zeros(128, dtype=torch.uint8, device="cuda")
                if rank == 0:
                    t2.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
                dist.broadcast(t2, 0)
                nid2 = bytes(t2.cpu().numpy())
            serve_model = RecModel(cfg, seed=1, max_batch=max(ds), streams=m_streams, device=local,
                                   l2_persist_bytes=l2p, rank=rank, world=world, nccl_id=nid2)
        res = gradient_search(evaluate, ms, ds, noise=0.02)
        sla = {"sla_ms": cfg.sla_ms, "percentile": "p95 (nearest rank)",
               "lambda_star_qps": res["qps"], "policy": {"streams": res["m"], "max_batch": res["d"]},
               "alg1_path": res["path"], "alg1_evaluated": res["evaluated"],
               "queries_per_probe": args.sla_queries * world,
               "probes_at_best": probes_all.get(f"m{res['m']}_d{res['d']}"),
               "mode": "rec_serve real clock, Poisson arrivals, lognormal sizes (R13), split/fuse, "
                       "device-synth inputs, replica dispatch q mod G; Alg. 1 gradient search over "
                       "(streams, max_batch)"}

    # dense stages at the serving batch d: back-to-back launches on one stream (CUDA events)
    fb_i = sum(2 * x * y for x, y in zip(cfg.bottom[:-1], cfg.bottom[1:]))
    wt_i = [cfg.top_in] + list(cfg.top)
    ft_i = cfg.tasks * sum(2 * x * y for x, y in zip(wt_i[:-1], wt_i[1:]))
    tb_d = model.rec_bench_mlp(0, d, 50) if fb_i else 0.0
    ti_d = model.rec_bench_mlp(2, d, 50)
    tt_d = model.rec_bench_mlp(1, d, 50)
    mlp_serving = {"batch": d,
                   "bottom": ({"us": 1e3 * tb_d, "tflops": fb_i * d / (tb_d * 1e-3) / 1e12}
                              if fb_i else None),
                   "top": {"us": 1e3 * (tt_d - ti_d),
                           "tflops": ft_i * d / ((tt_d - ti_d) * 1e-3) / 1e12},
                   "join_us": 1e3 * ti_d,
                   "measured": "rec_bench_mlp at the serving batch d: 50 back-to-back launches of "
                               "each stage on one stream (CUDA events)"}
    mlp_step_tflops = mlp_flops_per_item(cfg) * tot_items / (ms_max * 1e-3) / 1e12 / world

    # MLP tensor-pipe utilisation at a large batch (north_star "MLP TC util"): the same MLP
    # stacks in a second handle with max_batch = --mlp-batch (tiny tables: SLS not involved)
    mlp_large = mlp_large_batch(cfg, args.mlp_batch, local) if args.mlp_batch > 0 and rank == 0 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        ob = oracle_baseline(args.config, args.cpu_items, args.cpu_jobs_per_core, cores)
        mean_q = float(sizes.mean())
        cpu = {"value": ob["items_per_s"] / mean_q, "unit": "QPS", "cores": cores, "kind": "oracle",
               "cpu_model": cpu_model(), "value_1core": ob["items_per_s_1core"] / mean_q,
               "sample": f"{ob['items']} items of {cfg.name} ({cores * args.cpu_jobs_per_core} jobs x "
                         f"{args.cpu_items} items; fp64 oracle forward, {ob['cpu_s']:.1f} CPU-s, "
                         f"{ob['wall_s']:.2f} s wall on a warm {cores}-process pool; inputs generated "
                         f"before the timed map)",
               "items_per_s": ob["items_per_s"], "items_per_s_1core": ob["items_per_s_1core"]}

    models = {}
    for name in [x for x in args.per_model.split(",") if x and x != args.config]:
        models[W.SHORT[name].name] = per_model(name, args, rank, world, dist, local, hbm_peak)

    if rank == 0:
        line = {
            "metric": BASELINE_METRIC, "value": value, "unit": "QPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 (SLS) + bf16 (MLP, fp32 accumulate)", "data": "synthetic",
            "config": {"workload": cfg.name, "max_batch_d": d, "l2_persist_mb": args.l2_persist_mb, "tables": cfg.num_tables,
                       "rows": cfg.rows, "dim": cfg.dim, "pooling": cfg.pooling_lo,
                       "items_per_s": tot_items / (ms_max * 1e-3), "queries_per_step": tot_q / args.steps / world,
                       "mean_query_items": float(sizes.mean()), "parallelism": f"replicas x{world}",
                       "streams_per_gpu": m_streams, "pipeline_lanes": args.pipe,
                       "l2": "inputs larger than L2 (1.28 GB tables, uniform random rows per step)",
                       "value_is": "saturation QPS (burst trace); see sla"},
            "roofline": {"bound": "hbm", "kernel": "k_sls", "achieved": sls_gbs, "peak": hbm_peak,
                         "unit": "GB/s", "frac": (sls_gbs / hbm_peak) if sls_gbs else None,
                         "traffic": traffic, "traffic_source": "profiles/sls_traffic.json (ncu --set full)",
                         "algorithmic_bytes_per_launch": b2b_bytes / max(b2b_n, 1), "peak_kind": peak_kind,
                         "bytes_per_item": sls_bytes_per_item(cfg, synth=True),
                         "avg_launch_us": 1e3 * b2b_ms / max(b2b_n, 1),
                         "measured": f"rec_bench_sls: the first {b2b_n} batches of the timed sequence, "
                                     f"one launch each, back to back on one stream (distinct rows per "
                                     f"launch: no L2 reuse between launches) "
                                     f"(programmatic dependent launch: a launch's gathers overlap the "
                                     f"previous launch's drain, its stores wait for it; CUDA events on "
                                     f"that stream, time / launches)",
                         "serialized": {"achieved": sls_gbs_ser,
                                        "frac": (sls_gbs_ser / hbm_peak) if sls_gbs_ser else None,
                                        "avg_launch_us": 1e3 * ser_ms / max(b2b_n, 1),
                                        "measured": "same batches, plain launches back to back (no "
                                                    "overlap; each launch's ramp, drain and launch gap "
                                                    "included)"},
                         "isolated": {"achieved": sls_gbs_isolated,
                                      "frac": (sls_gbs_isolated / hbm_peak) if sls_gbs_isolated else None,
                                      "avg_launch_us": 1e3 * sls_ms / max(sls_n, 1), "launches": sls_n,
                                      "measured": f"CUDA event nodes around the SLS node inside the "
                                                  f"step graph, {rsteps} single-stream steps (includes "
                                                  f"launch gap and ramp of a lone launch)"},
                         "caller_index": caller,
                         "in_step_aggregate": {
                             "achieved": sls_bytes_per_item(cfg, synth=True) * tot_items / (ms_max * 1e-3) / 1e9 / world,
                             "frac": sls_bytes_per_item(cfg, synth=True) * tot_items / (ms_max * 1e-3) / 1e9 / world / hbm_peak,
                             "measured": "per GPU: SLS algorithmic bytes of all timed steps / timed region "
                                         "/ ranks (all kernels of the step running on co-located streams)"}},
            "mlp": {"bound": "tensor", "achieved_tflops": gemm_tf, "peak": bf16_peak,
                    "frac": (gemm_tf / bf16_peak) if gemm_tf else None, "flops_per_item": mlp_flops_per_item(cfg),
                    "launches": gemm_n, "ms": gemm_ms,
                    "measured": "per-launch CUDA events in the single-stream pass (batches <= d: "
                                "latency-bound)", "serving_batch": mlp_serving,
                    "in_step_aggregate": {"tflops_per_gpu": mlp_step_tflops,
                                          "frac": mlp_step_tflops / bf16_peak},
                    "large_batch": mlp_large},
            "breakdown_us_per_batch_single_stream": {
                "gen": 1e3 * gen_ms / rsteps, "sls": 1e3 * sls_ms / rsteps,
                "gemm": 1e3 * gemm_ms / rsteps, "interact": 1e3 * int_ms / rsteps},
            "gpu_launches": int(launches),
            "host_submit_us_per_step": 1e6 * host_submit_s / args.steps,
            "host_submit_breakdown_per_step": host_prof,
            "clocks": clk.summary(t_region0, t_region1),
            "e2e": e2e,
            "sla": sla,
            "cpu_baseline": cpu,
            "per_model": models,
        }
        if sla:
            sla["saturation_ge_lambda_star"] = bool(value >= LAMBDA_TOL * sla["lambda_star_qps"])
        if cfg.arch == W.ARCH_MTWND:
            # one-hot lookups move ~1 KB per item; the task towers (7.4 MFLOP per item) dominate:
            # report the tensor roofline of the tower GEMMs first, the SLS one beside it
            top = mlp_serving["top"]
            line["roofline_sls"] = line["roofline"]
            line["roofline"] = {
                "bound": "tensor", "kernel": "k_gemm_tc (task towers)", "achieved": top["tflops"],
                "peak": bf16_peak, "unit": "TFLOP/s", "frac": top["tflops"] / bf16_peak,
                "traffic": None, "peak_kind": peak_kind,
                "flops_per_item": ft_i, "avg_launch_us": top["us"],
                "measured": mlp_serving["measured"] + "; towers = (concat + towers) - concat",
                "in_step_aggregate": line["mlp"]["in_step_aggregate"]}
        print(json.dumps(line), flush=True)
    model.close()
    if world > 1:
        dist.destroy_process_group()


def run_sharded(args):
    """Model-parallel serving (BASELINE configs[2]: RMC2 "table-wise sharded across 8 x B200 with
    all-to-all"): the embedding tables are split over the G ranks (table-wise: T/G tables per
    rank), every rank runs the SAME global batches on m co-located stream slots, the all-to-all
    of pooled vectors and the CTR all-gather are fused into the chain as peer stores over
    NVLink with per-slot epoch flags (dist.cu), several global batches in flight per rank.
    value = queries of the global batches / device time (counted once; scaling "strong");
    sla = lambda* of rec_serve with the deterministic global dispatcher (reading R31)."""
    import torch
    import torch.distributed as dist
    from paper_2203_07424_b200 import (RecModel, nccl_unique_id, REC_SHARD_TABLE, REC_SHARD_ROW)
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = W.SHORT[args.config]
    d = args.batch
    m_streams = default_streams(args, args.config)
    t = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0)
    shard = REC_SHARD_TABLE if args.shard == "table" else REC_SHARD_ROW
    model = RecModel(cfg, seed=1, max_batch=d, streams=m_streams, device=local, shard=shard, rank=rank,
                     world=world, nccl_id=bytes(t.cpu().numpy()))
    hbm_peak, bf16_peak, peak_kind = peaks()
    clk = ClockSampler(local).__enter__()
    sat = saturation(model, cfg, d, m_streams, args.steps, args.warmup, args.step_batches,
                     args.queries, rank, world, dist, sharded=True)
    clk.__exit__(None, None, None)
    ms_max, items, queries = sat["ms_max"], sat["items"], sat["queries"]
    value = queries / (ms_max * 1e-3)
    # e2e: the same global batches with pinned HOST inputs (rec_query_async on the slots: H2D of
    # the global batch's inputs on every rank) and the gathered CTRs read back
    batches, nb = sat["batches"], sat["nb"]
    host = []
    for b in range(min(nb, 32)):
        ind, off, dense = model.rec_gen_batch(batches[b])
        host.append((torch.from_numpy(dense).pin_memory(), torch.from_numpy(ind).pin_memory(),
                     torch.from_numpy(off).pin_memory(), int(off[-1]), int(batches[b][:, 2].sum()),
                     sat["done_b"][b]))
    outs = [torch.empty(d).pin_memory() for _ in range(m_streams)]
    nb_e2e = max(1, args.e2e_steps) * args.step_batches
    for i in range(2 * m_streams):
        h = host[i % len(host)]
        model.rec_query_async(i % m_streams, h[0], h[1], h[2], h[3], h[4], outs[i % m_streams])
    for k in range(m_streams):
        model.rec_sync(k)
    from paper_2203_07424_b200 import rec_shard_plan

    def h2d_bytes(h):  # what rec_query_async copies on this rank: offsets, the local tables'
        B = h[4]       # indices, the own block's dense rows (include/rec.h)
        pl = rec_shard_plan([cfg.rows] * cfg.num_tables, world, rank, shard, B)
        off = h[2].numpy()
        nidx = int(off[(pl["t0"] + pl["t_local"]) * B]) - int(off[pl["t0"] * B])
        return 4 * (off.size + nidx + pl["items"] * cfg.dense_dim)
    hb = [h2d_bytes(h) for h in host]
    dist.barrier()
    t0 = time.perf_counter()
    q_e2e = h2d = d2h = 0
    for i in range(nb_e2e):
        h = host[i % len(host)]
        model.rec_query_async(i % m_streams, h[0], h[1], h[2], h[3], h[4], outs[i % m_streams])
        q_e2e += h[5]
        h2d += hb[i % len(host)]
        d2h += 4 * h[4]
    for k in range(m_streams):
        model.rec_sync(k)
    wall = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    dist.all_reduce(wall, op=dist.ReduceOp.MAX)
    sla = None
    if args.sla_queries > 0:
        n = int(max(30000, 1.5 * value))
        lam, pr = sla_search(model, cfg, world, rank, dist, m_streams, d, 0.5 * value, n, cfg.sla_ms,
                             replicated=True)
        sla = {"sla_ms": cfg.sla_ms, "percentile": "p95 (nearest rank)", "lambda_star_qps": lam,
               "policy": {"streams": m_streams, "max_batch": d,
                          "fusion": "deterministic global dispatcher, tau = SLA/50 (R31)"},
               "queries_per_probe": n, "probes": pr,
               "saturation_ge_lambda_star": bool(value >= LAMBDA_TOL * lam),
               "mode": "rec_serve real clock on every rank (same trace, same batches), Poisson "
                       "arrivals, lognormal sizes; p95 of rank 0's completions"}
    per_gpu = sls_bytes_per_item(cfg, synth=True) * items / (ms_max * 1e-3) / 1e9 / world
    if rank == 0:
        line = {
            "metric": BASELINE_METRIC, "value": value, "unit": "QPS",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 (SLS) + bf16 (MLP, fp32 accumulate)", "data": "synthetic",
            "config": {"workload": cfg.name, "max_batch_d": d, "tables": cfg.num_tables,
                       "rows": cfg.rows, "dim": cfg.dim, "pooling": cfg.pooling_lo,
                       "parallelism": f"{args.shard}-wise sharding x{world}, {m_streams} async slots "
                                      f"(all-to-all + CTR all-gather fused as peer stores over NVLink)",
                       "items_per_s": items / (ms_max * 1e-3), "step_batches": args.step_batches,
                       "l2": "inputs larger than L2 (tables >> 126 MB, uniform random rows)",
                       "value_is": "saturation QPS of the global batch stream"},
            "roofline": {"bound": "hbm", "kernel": "k_sls_synth (sharded, peer stores)", "achieved": per_gpu,
                         "peak": hbm_peak, "unit": "GB/s", "frac": per_gpu / hbm_peak, "traffic": None,
                         "peak_kind": peak_kind,
                         "measured": "per-GPU share of the SLS algorithmic bytes / the timed region "
                                     "(the chain also runs the exchange waits and the dense part)"},
            "gpu_launches": int(sat["launches"]),
            "clocks": clk.summary(sat["t0"], sat["t1"]),
            "e2e": {"value": q_e2e / float(wall[0]), "unit": "QPS",
                    "h2d_bytes_per_step": int(h2d / max(args.e2e_steps, 1)),
                    "d2h_bytes_per_step": int(d2h / max(args.e2e_steps, 1)), "steps": args.e2e_steps,
                    "api": "rec_query_async with pinned host inputs on the async slots, max wall over ranks"},
            "sla": sla,
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    model.close()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--per-model", default="rmc2,rmc3,mtwnd",
                    help="other workloads reported in the line's per_model block ('' = none)")
    ap.add_argument("--pm-steps", type=int, default=6)
    ap.add_argument("--pm-step-batches", type=int, default=256)
    ap.add_argument("--pm-sla", type=int, default=1, help="lambda* for the per_model workloads")
    ap.add_argument("--step-batches", type=int, default=512,
                    help="fused batches per step (one serving round over the co-located streams)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="rmc1", choices=list(W.SHORT))
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--streams", type=int, default=0,
                    help="co-located streams m (0 = per workload: 32 for RMC3, whose dense chain "
                         "is latency-bound (16 -> 32: +16 %), else 16)")
    ap.add_argument("--submit", default="batch", choices=["batch", "python"])
    ap.add_argument("--shard", default="replica", choices=["replica", "table", "row"],
                    help="N > 1: model-parallel embedding sharding instead of replicas")
    ap.add_argument("--pipe", type=int, default=0,
                    help="S-D pipeline lanes (rec_set_pipeline) for the timed region; 0 = slot graphs")
    ap.add_argument("--roofline-steps", type=int, default=1000)
    ap.add_argument("--sls-batches", type=int, default=1000, help="batches in the back-to-back SLS pass")
    ap.add_argument("--caller-batches", type=int, default=48,
                    help="distinct device-resident batches in the caller-index SLS pass (0 = off)")
    ap.add_argument("--queries", type=int, default=40000)
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--sla-queries", type=int, default=100000, help="Poisson queries per probe per GPU")
    ap.add_argument("--l2-persist-mb", type=int, default=0,
                    help="L2 persisting window over the hot row prefix of the tables (MB, 0 = off)")
    ap.add_argument("--max-batch-search", type=int, default=0,
                    help="largest fusion batch d in the Alg. 1 search (0 = per-config default: "
                         "1024 for RMC1 and tiny, 4096 otherwise)")
    ap.add_argument("--fusion-timeout-ms", type=float, default=0.0,
                    help="serving policy tau: a partial batch waits up to tau for more queries (R15)")
    ap.add_argument("--cpu-items", type=int, default=128, help="items per cpu_baseline oracle job")
    ap.add_argument("--cpu-jobs-per-core", type=int, default=3)
    ap.add_argument("--mlp-batch", type=int, default=65536, help="large-batch MLP TC probe (0 = off)")
    ap.add_argument("--ref-items", type=int, default=64)
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="reference arm: target wall time of the K timed steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    args.streams_auto = args.streams == 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torch.distributed.run
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
               str(port), os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    if args.impl == "reference":
        run_reference(args)
    elif args.shard != "replica" and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        run_sharded(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
