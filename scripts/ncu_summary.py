"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) per kernel.

usage: python scripts/ncu_summary.py launches.csv [--last N]
Prints count, total and mean duration per kernel name (mean over the last N launches of
each kernel when --last is given, i.e. the timed region of a bench run).
"""
import argparse
import collections
import csv


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    out = []
    for r in data:
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        out.append((r[ki], v))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--last", type=int, default=0)
    a = ap.parse_args()
    agg = collections.defaultdict(list)
    for k, v in load(a.csv):
        agg[k.split("(")[0][:70]].append(v)
    tot_all = 0.0
    lines = []
    for k, v in agg.items():
        sel = v[-a.last:] if a.last else v
        tot_all += sum(sel)
        lines.append((sum(sel), len(v), sum(sel) / len(sel), k))
    print(f"{'kernel':70s} {'n':>6s} {'sum_us':>10s} {'mean_us':>9s} {'share':>6s}")
    for s, n, m, k in sorted(lines, reverse=True):
        print(f"{k:70s} {n:6d} {s:10.1f} {m:9.2f} {100 * s / tot_all:5.1f}%")


if __name__ == "__main__":
    main()
