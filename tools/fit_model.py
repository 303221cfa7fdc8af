"""Fit the B200 cost model to measured latencies and regenerate
the selection table (the reference's calibrate(), calibrate.cpp:67-181, and
selection_table(), sweep.cpp:229-287, for the B200 executor).

    python tools/fit_model.py [--out profiles/b200_model_fit_r02.json]
                              [--table profiles/b200_selection_table_r02.md]
                              [--latency CSV ...] [--sweep CSV ...]

Measurements (device time per collective, back to back, explicit plans, one
caller stream, ranks co-resident on one B200):
  * tools/latency.cpp CSVs (api=plan rows; 4 KiB - 1 MiB; no Python in the loop);
  * bench.py --sweep --api plan CSVs, chunks >= 4 MiB only (below, the
    Python-driven loop is host-bound and would fit the host, not the device).
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2511_06605_b200 as cc  # noqa: E402

MODEL_IMPLS = {"sm", "pcpy", "b2b", "bcst", "swap", "prelaunch_pcpy", "prelaunch_b2b", "prelaunch_bcst",
               "prelaunch_swap"}
DEFAULT_LATENCY = ["profiles/latency_r02_n8_final.csv", "profiles/latency_r02_n4_final.csv",
                   "profiles/latency_r02_n2_final.csv"]
DEFAULT_SWEEP = ["profiles/sweep_r02_plan_n8_final.csv", "profiles/sweep_r02_plan_n4_final.csv",
                 "profiles/sweep_r02_plan_n2_final.csv"]
SWEEP_MIN = 4 << 20


def load_rows(latency, sweep):
    rows, sources = [], []
    for path in latency:
        full = os.path.join(ROOT, path)
        if not os.path.exists(full):
            continue
        n = 2 if "_n2" in path else 4 if "_n4" in path else 8
        sources.append(path)
        for r in csv.DictReader(open(full)):
            if r.get("api") != "plan" or r.get("impl") not in MODEL_IMPLS:
                continue
            if r.get("collective") not in ("allgather", "alltoall"):
                continue
            rows.append((r["collective"], r["impl"], int(r["size_bytes"]), n, float(r["device_us_b2b"]) * 1e3))
    for path in sweep:
        full = os.path.join(ROOT, path)
        if not os.path.exists(full):
            continue
        sources.append(path)
        for r in csv.DictReader(open(full)):
            if r.get("impl") not in MODEL_IMPLS or r.get("gpus") != "1" or not r.get("total_ns"):
                continue
            s = int(r["size_bytes"])
            if s < SWEEP_MIN:
                continue
            rows.append((r["collective"], r["impl"], s, int(r["ranks"]), float(r["total_ns"])))
    return rows, sources


def measured_grid(rows):
    """(kind, n) -> {s: {impl: ns}}"""
    g = {}
    for kind, impl, s, n, ns in rows:
        g.setdefault((kind, n), {}).setdefault(s, {})[impl] = ns
    return g


def selection_table(model, rows):
    """Per (collective, n, s): the model's winner, the measured winner, and
    whether they agree within the reference's tolerance: the same winner at
    this size or one grid step away (acceptance.cpp:85-87), or a measured
    time of the model's pick within 10% of the best (a tie on the device)."""
    out = []
    for (kind, n), by_s in sorted(measured_grid(rows).items()):
        sizes = sorted(by_s)
        mwin = {s: min(by_s[s], key=by_s[s].get) for s in sizes}
        for i, s in enumerate(sizes):
            cands = by_s[s]
            pick = min(cands, key=lambda c: model.predict_ns(kind, c, s, n))
            near = {mwin[sizes[j]] for j in (i - 1, i, i + 1) if 0 <= j < len(sizes)}
            tie = cands[pick] <= 1.10 * cands[mwin[s]]
            out.append({"collective": kind, "n": n, "s": s, "model": pick, "measured": mwin[s],
                        "measured_ns": round(cands[mwin[s]]), "model_pick_measured_ns": round(cands[pick]),
                        "predicted_ns": round(model.predict_ns(kind, pick, s, n)),
                        "match": pick == mwin[s], "within_one_step": pick in near or tie})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "b200_model_fit_r02.json"))
    ap.add_argument("--table", default=os.path.join(ROOT, "profiles", "b200_selection_table_r02.md"))
    ap.add_argument("--latency", nargs="*", default=DEFAULT_LATENCY)
    ap.add_argument("--sweep", nargs="*", default=DEFAULT_SWEEP)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--iterations", type=int, default=20000)
    args = ap.parse_args()
    rows, sources = load_rows(args.latency, args.sweep)
    default = cc.Model()
    model, residual, report = cc.Model.fit(rows, seed=args.seed, iterations=args.iterations)
    _, default_residual, _ = cc.Model.fit(rows, seed=args.seed, iterations=0)
    table = selection_table(model, rows)
    res = {"sources": sources, "measurements": len(rows), "seed": args.seed, "iterations": args.iterations,
           "default_params": default.p.as_dict(), "default_residual": default_residual,
           "params": model.p.as_dict(), "residual": residual, "report": report,
           "table": table, "within_one_step": sum(r["within_one_step"] for r in table), "rows": len(table)}
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    with open(args.table, "w") as f:
        f.write("# B200 selection table from the fitted cost model (tools/fit_model.py)\n\n")
        f.write(f"Fitted to {len(rows)} measurements ({', '.join(sources)}); seed {args.seed}, "
                f"{args.iterations} hill-climb steps; residual {residual:.4f} (defaults: {default_residual:.4f}).\n\n")
        f.write("| param | default | fitted |\n|---|---|---|\n")
        for k, v in model.p.as_dict().items():
            f.write(f"| {k} | {default.p.as_dict()[k]:.4g} | {v:.4g} |\n")
        f.write("\n| collective | n | s | model winner | measured winner | model pick measured µs | best µs "
                "| predicted µs | agrees (one step / tie) |\n|---|---|---|---|---|---|---|---|---|\n")
        for r in table:
            f.write(f"| {r['collective']} | {r['n']} | {r['s']} | {r['model']} | {r['measured']} | "
                    f"{r['model_pick_measured_ns'] / 1e3:.1f} | {r['measured_ns'] / 1e3:.1f} | "
                    f"{r['predicted_ns'] / 1e3:.1f} | {'yes' if r['within_one_step'] else 'NO'} |\n")
        f.write("\nBoundary report of the fit (calibrate.cpp:44-62 rule):\n\n```\n" + report + "```\n")
    print(f"residual {default_residual:.4f} -> {residual:.4f}; {res['within_one_step']}/{len(table)} sizes agree")


if __name__ == "__main__":
    main()
