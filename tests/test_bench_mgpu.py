"""Host logic of the multi-GPU bench arm (bench_mgpu.py) on CPU: the seeded
chunk patterns every process rebuilds, the cross-rank consensus helpers over
gloo (world size 2), and the watchdog's partial line."""
import json
import os
import socket
import subprocess
import sys
import textwrap
import traceback

import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench_mgpu as bm  # noqa: E402


@pytest.mark.parametrize("kind", ["allgather", "alltoall"])
@pytest.mark.parametrize("n", [2, 3, 8])
def test_expectations_match_the_collective_definition(kind, n):
    s = 96
    in_bytes = s if kind == "allgather" else n * s
    sends = [torch.zeros(in_bytes, dtype=torch.uint8) for _ in range(n)]
    expects = [torch.zeros(n * s, dtype=torch.uint8) for _ in range(n)]
    bm.fill_and_expect(kind, s, n, list(range(n)), sends, expects, "cpu")
    for j in range(n):
        for i in range(n):
            src = sends[i][:s] if kind == "allgather" else sends[i][j * s:(j + 1) * s]
            # compiler.cpp:119-126: rank i's chunk (AG) / chunk j of rank i (AA) lands in slot i of rank j
            assert torch.equal(expects[j][i * s:(i + 1) * s], src), (kind, n, i, j)
    # every (rank, chunk) pattern is distinct: a misrouted chunk cannot pass parity
    chunks = {bytes(sends[i][j * s:(j + 1) * s].tolist()) for i in range(n)
              for j in range(1 if kind == "allgather" else n)}
    assert len(chunks) == n * (1 if kind == "allgather" else n)


def test_seeds_distinct_across_sizes_kinds_and_ranks():
    seen = set()
    for kind in ("allgather", "alltoall"):
        for s in [4096 << (2 * k) for k in range(10)]:
            for i in range(8):
                for j in range(8 if kind == "alltoall" else 1):
                    seen.add(bm.seed_of(kind, s, i, j))
    assert len(seen) == 10 * 8 + 10 * 64


def _free_port():
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    p = sk.getsockname()[1]
    sk.close()
    return p


def _consensus_worker(rank, world, port, q):
    try:
        import torch.distributed as dist

        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        r = {
            "all_true_mixed": bm.all_true(rank == 0),
            "all_true_all": bm.all_true(True),
            "max": bm.max_all(float(rank) + 0.5),
            "from0": bm.from_rank0({"impl": f"from-{rank}"}),
        }
        dist.destroy_process_group()
        q.put((rank, r))
    except Exception:  # noqa: BLE001
        q.put((rank, traceback.format_exc()))


def test_consensus_helpers_over_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_consensus_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank in (0, 1):
        r = res[rank]
        assert isinstance(r, dict), r
        assert r["all_true_mixed"] is False  # one rank's failure drops the plan everywhere
        assert r["all_true_all"] is True
        assert r["max"] == 1.5  # max over ranks
        assert r["from0"] == {"impl": "from-0"}  # every rank runs rank 0's choice


@pytest.mark.parametrize("phase,code,value", [("alltoall sm s=8 timing", 1, None),
                                              ("experiments sm_peer_tma alltoall", 0, None),
                                              ("nccl alltoall", 0, 700.0)])
def test_watchdog_prints_the_line_and_exits(phase, code, value):
    prog = textwrap.dedent(f"""
        import sys, time
        sys.path.insert(0, {ROOT!r})
        import bench_mgpu as bm
        line = {{"metric": "m", "value": {value!r}, "config": {{}}, "details": {{"impl_trials": {{
            "sm": {{"ms": 0.2, "busbw_gbs": 300.0}}, "pcpy": {{"error": "x"}}, "b2b": {{"ms": 0.1, "busbw_gbs": 600.0}}}}}}}}
        bm.STATE["phase"] = {phase!r}
        bm.Watchdog(0.2, 0, lambda: line)
        time.sleep(30)
    """)
    r = subprocess.run([sys.executable, "-c", prog], capture_output=True, text=True, timeout=60)
    assert r.returncode == code, r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    if code == 1:  # hung before the headline: best trial so far, flagged
        assert out["value"] == 600.0 and out["details"]["impl"].startswith("b2b")
        assert "watchdog" in out["error"]
    elif value is not None:  # hung after the headline: it stands, the phase is named
        assert out["value"] == value and "nccl" in out["error"]
    else:  # hung in an experiment: the main line stands
        assert out["experiments"]["hung"] == phase and "error" not in out
