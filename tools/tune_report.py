"""Run cecoll_tune on one B200 (n co-resident ranks) and print the installed
table, every candidate's device time per size, and the static selector's pick
beside the measured winner.   python tools/tune_report.py [n] [max_chunk]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_06605_b200 as cc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cap = int(float(sys.argv[2])) if len(sys.argv) > 2 else 64 << 20
comms = cc.Comm.init_all([0] * n)
stream = torch.cuda.Stream()
cc.tune(comms, max_chunk=cap, streams=stream)
rep = comms[0].tune_report()
rows = []
for (kind, s), v in sorted(rep.items()):
    best = min((t, i) for i, t in v["us"].items() if t > 0)
    static = cc.select(kind, s, n, 1)
    rows.append({"kind": kind, "s": s, "winner": v["winner"], "fastest": best[1], "static": static,
                 "static_over_winner": round(v["us"][static] / v["us"][v["winner"]], 3), "us": v["us"]})
print(json.dumps({"ranks": n, "max_chunk": cap, "table": [f"{k} {s} {i}" for k, s, i in comms[0].tuned_table()],
                  "rows": rows}, indent=1))
cc.destroy_all(comms)
