"""The reference's simulator re-run with B200-measured phase latencies.

ANALYSIS INFRASTRUCTURE: tools/phase_probe.cu measures the
cost-model parameters of cost_model.hpp:14-33 on a B200 (profiles/
b200_cost_model.conf); this script feeds them to the reference's own
simulate() (oracle/_ref/libdmasim_sim.so, built from proj/src/sim.cpp) and
compares the predictions with the measured latencies of the same command
programs (profiles/latency_r01_n8.csv, tools/latency.cpp) in the
control-dominated regime, then prints the selection table the reference's
model implies for B200 parameters.

    python oracle/b200_model.py > profiles/b200_model_vs_measured.md
"""
from __future__ import annotations

import csv
import ctypes as C
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SIM = os.path.join(HERE, "_ref", "libdmasim_sim.so")
IMPLS = {
    "allgather": ["pcpy", "bcst", "b2b", "prelaunch_pcpy", "prelaunch_bcst", "prelaunch_b2b"],
    "alltoall": ["pcpy", "swap", "b2b", "prelaunch_pcpy", "prelaunch_swap", "prelaunch_b2b"],
}
LINK = 900e9 / 7  # NVLink 5 per-GPU egress shared by 7 peers


def load():
    L = C.CDLL(SIM)
    L.sim_run.argtypes = [C.c_char_p, C.c_char_p, C.c_int64, C.c_int, C.c_char_p, C.c_double,
                          C.POINTER(C.c_double * 5)]
    return L


def simulate(L, kind, impl, s, n, cost_text, link=LINK):
    out = (C.c_double * 5)()
    rc = L.sim_run(kind.encode(), impl.encode(), s, n, cost_text.encode() if cost_text else None, link,
                   C.byref(out))
    if rc != 0:
        raise RuntimeError(f"simulate failed {kind} {impl} {s} {n}")
    return list(out)


def main():
    conf = os.path.join(ROOT, "profiles", "b200_cost_model.conf")
    cost = open(conf).read()
    L = load()
    meas = {}
    lat = os.path.join(ROOT, "profiles", "latency_r01_n8.csv")
    if os.path.exists(lat):
        for r in csv.DictReader(open(lat)):
            if r.get("api") == "eager":
                meas[(r["collective"], r["impl"], int(r["size_bytes"]))] = float(r["device_us_b2b"])
    now = {}
    lin = os.path.join(ROOT, "profiles", "latency_r01_n8_prelaunch_linear.csv")
    if os.path.exists(lin):  # explicit plans after recorded command lists / linear prelaunch bodies
        for r in csv.DictReader(open(lin)):
            if r.get("api") == "plan":
                now[(r["collective"], r["impl"], int(r["size_bytes"]))] = float(r["device_us_b2b"])
    n = 8
    print("# Reference simulator with B200-measured phase latencies vs measured\n")
    print(f"Cost model: `profiles/b200_cost_model.conf` (tools/phase_probe.cu); link {LINK / 1e9:.1f} GB/s "
          "per directed pair; n = 8. Measured: eager calls from C++ (tools/latency.cpp), 8 co-resident ranks.\n")
    print("The last column is the same program after the command-overhead work of round 1: plans replay one "
          "recorded CUDA graph per collective (DESIGN.md §3.7) and prelaunch bodies are two kernels (§3.4) "
          "(profiles/latency_r01_n8_prelaunch_linear.csv, explicit plans). The reference's model charges host "
          "control per command; recording removes exactly that term.\n")
    print("| collective | impl | s | simulated MI300X-default µs | simulated B200-params µs | measured eager µs "
          "| measured recorded / linear µs |")
    print("|---|---|---|---|---|---|---|")
    for kind in ("allgather", "alltoall"):
        for impl in IMPLS[kind]:
            for s in (4096, 65536):
                base = simulate(L, kind, impl, s, n, None, 64e9)[0] / 1e3
                b200 = simulate(L, kind, impl, s, n, cost)[0] / 1e3
                m = meas.get((kind, impl, s))
                r = now.get((kind, impl, s))
                print(f"| {kind} | {impl} | {s >> 10} KiB | {base:.1f} | {b200:.1f} | "
                      f"{'' if m is None else f'{m:.1f}'} | {'' if r is None else f'{r:.1f}'} |")
    print("\n## Selection under B200 parameters (simulated winner per size, n = 8)\n")
    print("| s | allgather | alltoall |")
    print("|---|---|---|")
    for k in range(10, 31, 2):
        s = 1 << k
        row = []
        for kind in ("allgather", "alltoall"):
            best = min(IMPLS[kind], key=lambda im: simulate(L, kind, im, s, n, cost)[0])
            row.append(best)
        print(f"| {s >> 10} KiB | {row[0]} | {row[1]} |")


if __name__ == "__main__":
    sys.exit(main())
