"""A caller's CUDA graph holding K collectives on per-rank streams (fork once,
join once), replayed back to back. Exploratory: run under `timeout`.
Usage: python tools/caller_graph_probe.py IMPL [K] [force]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 3 and sys.argv[3] == "force":
    os.environ["CECOLL_FORCE_REMOTE_SIGNALS"] = "1"
import numpy as np
import torch

import paper_2511_06605_b200 as cc
from oracle import oracle as ora

impl = sys.argv[1]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
n, s = 4, 16384 + 16
comms = cc.Comm.init_all([0] * n)
in_place = impl.endswith("swap")
hosts = [[ora.splitmix_pattern(n * s, r, 900 + it) for r in range(n)] for it in range(K)]
inputs = [[torch.from_numpy(hosts[it][r]).cuda() for r in range(n)] for it in range(K)]
sends = [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
recvs = sends if in_place else [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
outs = [[torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)] for _ in range(K)]
main = torch.cuda.Stream()
rs = [torch.cuda.Stream() for _ in range(n)]


def body():
    for r in range(n):
        rs[r].wait_stream(main)
    for it in range(K):
        for r in range(n):
            with torch.cuda.stream(rs[r]):
                sends[r].copy_(inputs[it][r])
        cc.all_to_all(comms, sends, recvs, s, impl=impl, streams=rs)
        for r in range(n):
            with torch.cuda.stream(rs[r]):
                outs[it][r].copy_(recvs[r])
    for r in range(n):
        main.wait_stream(rs[r])


with torch.cuda.stream(main):
    body()  # eager warm-up: plans built outside the capture
torch.cuda.synchronize()
print("eager ok", flush=True)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=main):
    body()
print("captured", flush=True)
bad = 0
for rep in range(3):
    for it in range(K):
        for t in outs[it]:
            t.zero_()
    torch.cuda.synchronize()
    g.replay()
    g.replay()  # back to back: the second replay overwrites outs with the same values
    torch.cuda.synchronize()
    for it in range(K):
        for r in range(n):
            want = np.concatenate([hosts[it][j][r * s:(r + 1) * s] for j in range(n)])
            if not np.array_equal(outs[it][r].cpu().numpy(), want):
                bad += 1
print(f"{impl} K={K} force={os.environ.get('CECOLL_FORCE_REMOTE_SIGNALS', '0')}: bad={bad} "
      f"async_error={comms[0].async_error()}", flush=True)
del g
cc.destroy_all(comms)
