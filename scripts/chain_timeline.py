"""Per-stage %globaltimer timeline of one fused-MLP CTA (diagnostic)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W
from paper_2203_07424_b200 import RecModel
names = {0: "entry", 1: "tmem+bars", 2: "tma0 issued", 3: "stage0 landed", 4: "L0 committed",
         5: "L1 committed", 8: "epi0 start", 9: "epi0 end", 10: "epi1 start", 11: "epi1 end", 15: "exit"}
for cfgname in sys.argv[1:] or ["rmc1"]:
    m = RecModel(W.SHORT[cfgname].with_(rows=1000), seed=1, max_batch=1024)
    for which in (0, 1):
        t = m.rec_debug_chain_timeline(which, 1024)
        base = t[0]
        row = {names[i]: round((t[i] - base) / 1e3, 2) for i in names if t[i]}
        row["event_us"] = round(t[14] / 1e3, 2)
        print(json.dumps({"cfg": cfgname, "mlp": ["bottom", "top"][which], "us": row}))
    m.close()
