"""The torchrun arm of bench.py (bench_mgpu.py) end to end on one GPU: two
processes share cuda:0 (NCCL is skipped there), every phase runs at reduced
sizes, and rank 0 prints one complete JSON line — the shape the driver's
round-end scaling run expects."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(600)
def test_torchrun_arm_prints_one_complete_line():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "5", "--warmup", "3", "--mgpu-sweep-max", "65536",
           "--interference-chunk", "1048576"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=550, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert "error" not in d, d.get("error")
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["parity_ok"] is True
    assert d["e2e"]["parity_ok"] is True and d["roofline"]["bound"] == "nvlink"
    assert all("ms" in v for v in d["details"]["impl_trials"].values()), d["details"]["impl_trials"]
    assert d["config"] == {"workload": d["config"]["workload"], "ranks": 8, "chunk_bytes": 8 << 20}
    assert all("graph_fallback" in v["plan"] for v in d["details"]["impl_trials"].values())
    rows = [row for row in d["sweep"]["rows"] if "skipped" not in row]
    assert rows and not any(row.get("errors") for row in rows)
    assert any(k.startswith("prelaunch") for row in rows for k in row.get("us", {}))  # the late pass ran
    assert d["interference"]["impls"] and d["sync_chain"]["cases"]
    assert "nvls_allgather" in d["experiments"]
