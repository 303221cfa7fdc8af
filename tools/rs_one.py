"""One reduce-scatter configuration, a few calls (for ncu captures):
python tools/rs_one.py [ranks] [chunk_bytes] [impl]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2511_06605_b200 as cc

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
s = int(sys.argv[2]) if len(sys.argv) > 2 else 64 << 20
impl = sys.argv[3] if len(sys.argv) > 3 else "sm"
count = s // 2
comms = cc.Comm.init_all([0] * n)
sends = [torch.randn(n * count, device="cuda").to(torch.bfloat16) for _ in range(n)]
recvs = [torch.empty(count, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
st = torch.cuda.Stream()
for _ in range(4):
    cc.reduce_scatter(comms, sends, recvs, count, dtype="bf16", op="sum", impl=impl, streams=st)
st.synchronize()
cc.destroy_all(comms)
print("ok", flush=True)
