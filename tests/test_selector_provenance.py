"""The B200 selector against the measured winner grid (winner_grid,
sweep.cpp:186-218): at every size of the committed one-GPU sweeps
(profiles/sweep_r01_plan_n{8,2}_recorded.csv, explicit plans) the
implementation cecoll_select picks for an out-of-place collective is within
10% of the fastest out-of-place implementation measured at that size — the
analogue of the reference's own check that its table matches the simulated
winners within tolerance (acceptance.cpp:85-87). CPU only: reads the CSVs."""
import csv
import os

import pytest

import paper_2511_06605_b200 as cc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1.10


def _grid(n):
    path = os.path.join(ROOT, "profiles", f"sweep_r01_plan_n{n}_recorded.csv")
    t = {}
    with open(path) as f:
        for r in csv.DictReader(f):
            if r.get("api") != "plan" or r["parity"] != "True" or r["impl"].endswith("swap"):
                continue  # in-place programs answer a different call
            t.setdefault((r["collective"], int(r["size_bytes"])), {})[r["impl"]] = int(r["total_ns"])
    return t


@pytest.mark.parametrize("n", [8, 2])
def test_selector_within_tolerance_of_measured_winner(n):
    grid = _grid(n)
    assert len(grid) >= 18
    worst = []
    for (kind, s), times in sorted(grid.items()):
        if s >= 1 << 30:
            continue  # 64 GiB per collective: bimodal between runs
        pick = cc.select(kind, s, n, 1)
        assert pick in times, (kind, s, pick)
        best = min(times.values())
        worst.append((times[pick] / best, kind, s, pick, min(times, key=times.get)))
        assert times[pick] <= TOL * best, (kind, s, pick, times)
    # the table in words: the SM path everywhere for all-gather, up to 32 MiB
    # for all-to-all, the driver's copies above
    assert cc.select("allgather", 1 << 28, n, 1) == "sm"
    assert cc.select("alltoall", 1 << 28, n, 1) == "b2b"
