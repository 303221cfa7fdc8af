"""Hardware timelines of one collective per implementation, in the
reference's trace-event format (load in chrome://tracing or Perfetto).

    python tools/trace_collective.py --kind alltoall --ranks 8 --chunk 1048576 --out gpurun_out/traces
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2511_06605_b200 as cc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="alltoall", choices=["allgather", "alltoall"])
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--chunk", type=int, default=1 << 20)
    ap.add_argument("--streams", default="per_rank", choices=["per_rank", "shared"])
    ap.add_argument("--impls", default="")
    ap.add_argument("--out", default="gpurun_out/traces")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    n, s = a.ranks, a.chunk
    comms = cc.Comm.init_all([0] * n)
    impls = a.impls.split(",") if a.impls else (
        ["sm", "pcpy", "b2b", "bcst", "prelaunch_pcpy", "prelaunch_b2b"] if a.kind == "allgather"
        else ["sm", "pcpy", "b2b", "swap", "prelaunch_pcpy", "prelaunch_b2b"])
    in_bytes = s if a.kind == "allgather" else n * s
    sends = [torch.randint(0, 255, (in_bytes,), dtype=torch.uint8, device="cuda") for _ in range(n)]
    recvs = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
    streams = ([torch.cuda.Stream() for _ in range(n)] if a.streams == "per_rank"
               else torch.cuda.current_stream())
    fn = cc.all_gather if a.kind == "allgather" else cc.all_to_all
    for impl in impls:
        out = sends if impl.endswith("swap") else recvs
        for _ in range(3):  # plans built and warm before tracing
            fn(comms, sends, out, s, impl=impl, streams=streams)
        torch.cuda.synchronize()
        with cc.Trace(comms[0]) as t:
            fn(comms, sends, out, s, impl=impl, streams=streams)
            torch.cuda.synchronize()
        path = os.path.join(a.out, f"trace_{a.kind}_{impl}_n{n}_s{s}.json")
        t.save(path)
        dev = [e["ts"] for e in t.events if e["pid"] >= 0]
        span = (max(dev) - min(dev)) if dev else 0.0
        print(f"{impl:15s} {len(t.events):5d} events, device span {span:9.1f} us -> {path}")
    cc.destroy_all(comms)


if __name__ == "__main__":
    main()
