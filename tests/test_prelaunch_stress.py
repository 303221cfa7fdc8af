"""Explicit prelaunch plans destroyed while armed, interleaved with eager
prelaunch calls on the same buffers — the sequence tools/latency.cpp runs per
(implementation, size). Round 2's first trigger-word version cancelled an
armed instance with a stream memory operation on a fresh stream, and a full
8-rank latency run hung in that sequence; cancels now raise a count in pinned
host memory (exec.cpp cancel_armed). Runs in a subprocess under a hard
timeout so a hang fails the test instead of the suite."""
import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import sys
    sys.path.insert(0, {root!r})
    import torch
    import paper_2511_06605_b200 as cc

    n = 8
    comms = cc.Comm.init_all([0] * n)
    per_rank = {per_rank}
    streams = [torch.cuda.Stream() for _ in range(n)] if per_rank else torch.cuda.Stream()
    bad = 0
    for rnd in range(3):
        for s in (4096, 16384, 65536, 262144):
            for kind in ("allgather", "alltoall"):
                impls = ["prelaunch_pcpy", "prelaunch_b2b"] + (["prelaunch_bcst"] if kind == "allgather"
                                                              else ["prelaunch_swap"])
                for impl in impls:
                    in_bytes = s if kind == "allgather" else n * s
                    sends = [torch.randint(0, 256, (in_bytes,), dtype=torch.uint8, device="cuda") for _ in range(n)]
                    swap = impl.endswith("swap")
                    recvs = [t.clone() for t in sends] if swap else [torch.zeros(n * s, dtype=torch.uint8,
                                                                                  device="cuda") for _ in range(n)]
                    torch.cuda.synchronize()
                    plan = cc.Plan(comms, kind, recvs if swap else sends, recvs, s, impl=impl)
                    for _ in range(3):
                        plan.launch(streams)
                    # armed now: no device-wide synchronisation before the
                    # destroy (cecoll.h cecoll_plan_disarm)
                    plan.destroy()  # armed: the cancel path
                    fn = cc.all_gather if kind == "allgather" else cc.all_to_all
                    for _ in range(3):
                        fn(comms, recvs if swap else sends, recvs, s, impl=impl, streams=streams)
                    torch.cuda.synchronize()
                    if not swap:  # 6 swaps restore the input; check the others against the definition
                        for i in range(n):
                            for j in range(n):
                                want = sends[i] if kind == "allgather" else sends[i][j * s:(j + 1) * s]
                                bad += not torch.equal(recvs[j][i * s:(i + 1) * s], want)
                    else:
                        bad += sum(not torch.equal(a, b) for a, b in zip(recvs, sends))
    cc.destroy_all(comms)
    print("bad", bad)
""")


@pytest.mark.timeout(400)
@pytest.mark.parametrize("per_rank", [False, True])
def test_destroy_armed_plans_between_eager_calls(per_rank):
    code = SCRIPT.format(root=ROOT, per_rank=per_rank)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=360, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "bad 0" in r.stdout, r.stdout[-2000:]
