"""Which chunks of a large co-resident all-to-all differ from their source?
   python tools/aa_big_check.py <s_bytes> [impl] [api]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_06605_b200 as cc  # noqa: E402

s = int(float(sys.argv[1]))
impl = sys.argv[2] if len(sys.argv) > 2 else "sm"
api = sys.argv[3] if len(sys.argv) > 3 else "plan"
kind = sys.argv[4] if len(sys.argv) > 4 else "alltoall"
n = 8
comms = cc.Comm.init_all([0] * n)
in_bytes = n * s if kind == "alltoall" else s
sends = [torch.randint(0, 256, (in_bytes,), dtype=torch.uint8, device="cuda") for _ in range(n)]
recvs = [torch.full((n * s,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(n)]
stream = torch.cuda.Stream()
torch.cuda.synchronize()
if api == "plan":
    plan = cc.Plan(comms, kind, sends, recvs, s, impl=impl)
    print(plan.info() if hasattr(plan, "info") else "")
for it in range(3):
    if api == "plan":
        plan.launch(stream)
    else:
        (cc.all_to_all if kind == "alltoall" else cc.all_gather)(comms, sends, recvs, s, impl=impl, streams=stream)
    stream.synchronize()
    bad = []
    for i in range(n):
        for j in range(n):
            src = sends[i][j * s:(j + 1) * s] if kind == "alltoall" else sends[i][:s]
            dst = recvs[j][i * s:(i + 1) * s]
            if not torch.equal(dst, src):
                d = (dst != src).nonzero()
                bad.append((i, j, int(d[0]), int(d[-1]), int(d.numel())))
    print(f"call {it}: {len(bad)} bad chunks", bad[:10])
    for t in recvs:
        t.fill_(0xA5)
    torch.cuda.synchronize()
print("async", [c.async_error() if hasattr(c, "async_error") else None for c in comms[:1]])
cc.destroy_all(comms)
