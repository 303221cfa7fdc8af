import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_06605_b200 as cc
from torch.profiler import ProfilerActivity, profile
n, s = 8, 65536
comms = cc.Comm.init_all([0] * n)
sends = [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
recvs = [torch.zeros(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
streams = [torch.cuda.Stream() for _ in range(n)]
for impl in ("b2b", "pcpy"):
    cc.all_to_all(comms, sends, recvs, s, impl=impl, streams=streams)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        cc.all_to_all(comms, sends, recvs, s, impl=impl, streams=streams)
        torch.cuda.synchronize()
    print(impl, [(e.key[:60], e.count) for e in prof.key_averages() if e.device_type.name == "CUDA" or "emcpy" in e.key][:20])
