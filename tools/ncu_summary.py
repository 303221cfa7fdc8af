"""Summarise one kernel of an ncu --set full report into profiles/*.json
(the fields bench.py reads: dram_bytes_per_launch, duration_us) plus every
raw metric with its unit.

  python tools/ncu_summary.py REPORT.ncu-rep OUT.json "capture description" [algorithmic_bytes]
"""
import csv
import io
import json
import subprocess
import sys


def main():
    rep, out, capture = sys.argv[1], sys.argv[2], sys.argv[3]
    alg = int(sys.argv[4]) if len(sys.argv) > 4 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    metrics = {h: [v, u] for h, u, v in zip(head, units, vals) if "__" in h}
    name = vals[head.index("Kernel Name")]

    def num(key, scale=1.0):
        v, u = metrics[key]
        f = float(v.replace(",", ""))
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
                "nsecond": 1e-3, "msecond": 1e3}.get(u, 1.0)
        return f * mult * scale

    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    d = {"kernel": "cecoll::" + name.split("::")[-1].split("(")[0], "capture": capture,
         "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
         "algorithmic_bytes_per_launch": alg, "duration_us": num("gpu__time_duration.sum"),
         "metrics": metrics}
    if alg:
        d["traffic_over_algorithmic"] = round((rd + wr) / alg, 4)
        d["achieved_gbs_cold"] = round(alg / (d["duration_us"] * 1e-6) / 1e9, 1)
    with open(out, "w") as f:
        json.dump(d, f, indent=1)
    print({k: v for k, v in d.items() if k != "metrics"})


if __name__ == "__main__":
    main()
