"""Diagnostic: pinned host -> device copy bandwidth on this box (the e2e leg's ceiling).
Copies of the e2e step's sizes (indices 3.28 MB, dense 1 MB, offsets 41 KB) on 1, 2 and 4
streams, CUDA events around 200 rounds."""
import json
import torch


def main():
    dev = torch.device("cuda", 0)
    sizes = {"indices": 10 * 80 * 1024 * 4, "dense": 1024 * 256 * 4, "offsets": 10 * 1024 * 4 + 4}
    out = {}
    for ns in (1, 2, 4):
        streams = [torch.cuda.Stream(dev) for _ in range(ns)]
        bufs = []
        for s in range(ns):
            bufs.append({k: (torch.empty(v, dtype=torch.uint8).pin_memory(),
                             torch.empty(v, dtype=torch.uint8, device=dev)) for k, v in sizes.items()})
        torch.cuda.synchronize()
        for rep in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for s in streams:
                s.wait_event(e0)
            n = 200
            for i in range(n):
                s = i % ns
                with torch.cuda.stream(streams[s]):
                    for k in sizes:
                        bufs[s][k][1].copy_(bufs[s][k][0], non_blocking=True)
            for s in streams:
                e = torch.cuda.Event()
                e.record(s)
                torch.cuda.current_stream().wait_event(e)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
        byt = n * sum(sizes.values())
        out[f"streams{ns}"] = round(byt / (ms * 1e-3) / 1e9, 2)
    big = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    dbig = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dbig.copy_(big, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
    out["single_256MB"] = round((256 << 20) / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)
    print(json.dumps({"h2d_GBps": out}))


if __name__ == "__main__":
    main()
