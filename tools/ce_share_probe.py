"""How do concurrent copy-engine streams share bandwidth on B200? (SURVEY §8
a15: the reference's run_flows / maxmin_rates, sim.cpp:28-63, 124-179, model
engine and link sharing as max-min fair fluid flows.) On one GPU the copy
engines carry host<->device traffic, so the probe starts k copies on k
streams at the same instant (every stream waits on one event) and records
each stream's completion time, then compares them with two models of the
link: max-min fair sharing (the reference's) and first-come-first-served.

   python tools/ce_share_probe.py [direction h2d|d2h|both]
"""
import json
import sys

import torch

MiB = 1 << 20


def run(sizes, direction):
    k = len(sizes)
    streams = [torch.cuda.Stream() for _ in range(k)]
    hosts = [torch.empty(s, dtype=torch.uint8, pin_memory=True) for s in sizes]
    devs = [torch.empty(s, dtype=torch.uint8, device="cuda") for s in sizes]
    dirs = [direction if direction != "both" else ("h2d" if i % 2 == 0 else "d2h") for i in range(k)]
    best = None
    for _ in range(5):
        torch.cuda.synchronize()
        go = torch.cuda.Event(enable_timing=True)
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        # hold every stream behind one event so the copies start together
        gate = torch.cuda.Stream()
        with torch.cuda.stream(gate):
            torch.cuda._sleep(2_000_000)  # ~1 ms of spin: every copy is queued before the gate opens
            go.record(gate)
        for i in range(k):
            streams[i].wait_event(go)
            with torch.cuda.stream(streams[i]):
                if dirs[i] == "h2d":
                    devs[i].copy_(hosts[i], non_blocking=True)
                else:
                    hosts[i].copy_(devs[i], non_blocking=True)
                ends[i].record(streams[i])
        torch.cuda.synchronize()
        t = [go.elapsed_time(e) for e in ends]
        if best is None or max(t) < max(best):
            best = t
    return dirs, best


def maxmin(sizes, bw):
    """Completion times (ms) of simultaneous flows sharing one link max-min fairly."""
    left = list(sizes)
    done = [None] * len(sizes)
    t = 0.0
    active = [i for i in range(len(sizes))]
    while active:
        rate = bw / len(active)
        step = min(left[i] for i in active) / rate
        t += step
        for i in list(active):
            left[i] -= rate * step
            if left[i] <= 1e-6:
                done[i] = t
                active.remove(i)
    return done


def fifo(sizes, bw):
    t, out = 0.0, []
    for s in sizes:
        t += s / bw
        out.append(t)
    return out


def main():
    direction = sys.argv[1] if len(sys.argv) > 1 else "h2d"
    res = {"direction": direction, "cases": []}
    # single-stream bandwidth of this direction (bytes per ms)
    _, t1 = run([256 * MiB], "h2d" if direction == "both" else direction)
    bw = 256 * MiB / t1[0]
    res["single_stream_gbs"] = round(bw / 1e6, 2)
    for sizes in ([64 * MiB] * 2, [64 * MiB] * 4, [64 * MiB] * 8, [256 * MiB] + [16 * MiB] * 3,
                  [16 * MiB] * 3 + [256 * MiB], [4 * MiB] * 8):
        dirs, t = run(sizes, direction)
        case = {"sizes_mib": [s // MiB for s in sizes], "dirs": dirs, "done_ms": [round(x, 3) for x in t]}
        if direction != "both":
            case["maxmin_ms"] = [round(x, 3) for x in maxmin(sizes, bw)]
            case["fifo_ms"] = [round(x, 3) for x in fifo(sizes, bw)]
            case["aggregate_gbs"] = round(sum(sizes) / max(t) / 1e6, 2)
        res["cases"].append(case)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
