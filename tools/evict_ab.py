"""A/B of the TMA mover's L2 policy by chunk size (run once per setting of
CECOLL_TMA_EVICT_FIRST): all-to-all and all-gather, SM path, 8 co-resident
ranks, device time per collective (median of 5 runs of 10)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_06605_b200 as cc  # noqa: E402

n = 8
comms = cc.Comm.init_all([0] * n)
st = torch.cuda.Stream()
tag = os.environ.get("CECOLL_TMA_EVICT_FIRST", "0")
for kind in ("alltoall", "allgather"):
    for mib in (2, 8, 32, 64, 128, 256):
        s = mib << 20
        ib = s if kind == "allgather" else n * s
        sends = [torch.empty(ib, dtype=torch.uint8, device="cuda") for _ in range(n)]
        recvs = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
        fn = cc.all_gather if kind == "allgather" else cc.all_to_all
        for _ in range(3):
            fn(comms, sends, recvs, s, impl="sm", streams=st)
        st.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(10):
                fn(comms, sends, recvs, s, impl="sm", streams=st)
            e1.record(st)
            st.synchronize()
            ts.append(e0.elapsed_time(e1) / 10)
        ts.sort()
        print(f"evict_first={tag} {kind} s={mib}MiB {ts[2] * 1e3:.1f} us", flush=True)
        del sends, recvs
        torch.cuda.empty_cache()
cc.destroy_all(comms)
