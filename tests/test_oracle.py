"""The oracle (plain-C restatement) pinned against the reference.

tests/golden/ was produced from the reference's own compile()/dump_program()/
static_metrics()/account_traffic()/verify_collective()/select_implementation()
(oracle/make_golden.py over oracle/_ref). When oracle/_ref is present (this
build container) the restatement is also compared with the reference live.
"""
import ctypes as C
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle as ora

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def O():
    return ora.Oracle()


@pytest.fixture(scope="module")
def programs():
    with open(os.path.join(GOLDEN, "programs.json")) as f:
        return json.load(f)


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def test_dump_metrics_traffic_match_reference(O, programs):
    checked = 0
    for e in programs["programs"]:
        p = O.compile(e["kind"], e["impl"], e["s"], e["n"])
        try:
            text = O.dump(p)
            assert sha(text.encode()) == e["dump_sha256"], (e["kind"], e["impl"], e["n"], e["s"])
            if "dump" in e:
                assert text == e["dump"]
            assert O.metrics(p) == e["metrics"]
            t, gr, gw = O.traffic(p, e["n"])
            assert t == e["traffic"]
            assert gr == e["per_gpu_read"] and gw == e["per_gpu_write"]
            if "verdict" in e:
                assert O.verify(p, trials=50, seed=3) == e["verdict"] == "ok"
            checked += 1
        finally:
            O.free(p)
    assert checked == len(programs["programs"]) == 540


def test_rejections_match_reference(O, programs):
    for r in programs["rejects"]:
        if r["accepted"]:
            p = O.compile(r["kind"], r["impl"], r["s"], r["n"])
            O.free(p)
        else:
            with pytest.raises(ValueError):
                O.compile(r["kind"], r["impl"], r["s"], r["n"])


def test_select_matches_reference(O):
    with open(os.path.join(GOLDEN, "select.json")) as f:
        table = json.load(f)
    for kind, rows in table.items():
        for size, name in rows:
            assert O.select(kind, size) == name, (kind, size)


def test_pattern_c_matches_numpy(O):
    for nbytes, rank, seed in [(1024, 0, 0), (4099, 3, 1), (17, 7, 0), (65536, 5, 0)]:
        assert np.array_equal(O.fill(nbytes, rank, seed), ora.splitmix_pattern(nbytes, rank, seed))


def test_byte_digests_match_reference(O):
    with open(os.path.join(GOLDEN, "digests.json")) as f:
        digests = json.load(f)
    for d in digests:
        orig, res = O.run(d["kind"], d["impl"], d["s"], d["n"], d["seed"])
        assert [sha(r.tobytes()) for r in res] == d["sha256"], d
        assert O.check(d["kind"], d["s"], d["n"], d["impl"].endswith("swap"), orig, res) == -1


def test_postcondition_checker_catches_corruption(O):
    orig, res = O.run("allgather", "pcpy", 1024, 4)
    assert O.check("allgather", 1024, 4, False, orig, res) == -1
    res[2][3 * 1024 + 5] ^= 1
    assert O.check("allgather", 1024, 4, False, orig, res) == 2 * 4 + 3


def _mutable(O, kind, impl, s, n):
    return O.compile(kind, impl, s, n)


def test_misrouted_copy_is_a_mismatch(O):
    # test_verifier.cpp:35-49: a copy 0->1 sent to slot 2 instead of slot 0
    p = O.compile("allgather", "pcpy", 1024, 4)
    try:
        prog = p.contents
        for qi in range(prog.nqueues):
            q = prog.queues[qi]
            for ci in range(q.ncmds):
                c = q.cmds[ci]
                if c.kind == 0 and c.src.gpu == 0 and c.dst.gpu == 1:
                    c.dst.offset = 2 * 1024
        assert O.verify(p, trials=20) == "mismatch"
    finally:
        O.free(p)


def test_random_interleavings_catch_misroute(O):
    # test_verifier.cpp:86-102: AA chunk 0 sent instead of chunk 3
    p = O.compile("alltoall", "pcpy", 1024, 4)
    try:
        prog = p.contents
        for qi in range(prog.nqueues):
            q = prog.queues[qi]
            for ci in range(q.ncmds):
                c = q.cmds[ci]
                if c.kind == 0 and c.src.gpu == 2 and c.dst.gpu == 3:
                    c.src.offset = 0
        assert O.verify(p, trials=200, seed=42) == "mismatch"
    finally:
        O.free(p)


def test_inplace_copy_exchange_is_a_hazard_swap_is_not(O):
    # test_verifier.cpp:51-84: two plain copies exchanging in place race; a Swap does not.
    p = O.compile("alltoall", "swap", 1024, 2)
    try:
        prog = p.contents
        assert prog.in_place == 1
        assert O.verify(p, trials=50) == "ok"
        # Rewrite into two queues of plain copies g -> 1-g on the in-place buffer.
        prog.nqueues = 2
        for g in (0, 1):
            q = prog.queues[g]
            q.gpu, q.engine, q.doorbell_count, q.ncmds = g, 0, 1, 2
            c = q.cmds[0]
            c.kind = 0
            c.src = ora.OraRef(g, 0, (1 - g) * 1024, 1024)
            c.dst = ora.OraRef(1 - g, 0, g * 1024, 1024)
            c.size = 1024
            s = q.cmds[1]
            s.kind = 3
            s.signal_target = g
        assert O.verify(p, trials=50) == "hazard"
    finally:
        O.free(p)


def test_reference_result_multithreaded(O):
    n, s = 8, 4096
    ins = [O.fill(n * s, r) for r in range(n)]
    outs1 = [np.zeros(n * s, np.uint8) for _ in range(n)]
    outs8 = [np.zeros(n * s, np.uint8) for _ in range(n)]
    O.reference_result("alltoall", s, n, ins, outs1, 1)
    O.reference_result("alltoall", s, n, ins, outs8, 8)
    assert O.check("alltoall", s, n, False, ins, outs1) == -1
    assert all(np.array_equal(a, b) for a, b in zip(outs1, outs8))


@pytest.mark.skipif(not os.path.exists(ora.REF_LIB), reason="oracle/_ref (the compiled reference) not built here")
def test_restatement_matches_live_reference(O):
    R = ora.Reference()
    rng = np.random.default_rng(0)
    for kind in ("allgather", "alltoall"):
        for impl in ora.IMPLS_FOR[kind]:
            for n in (2, 3, 6, 7, 9, 12, 16):
                s = int(rng.integers(1, 1 << 22))
                p = O.compile(kind, impl, s, n)
                try:
                    assert O.dump(p) == R.dump(kind, impl, s, n)
                    assert O.metrics(p) == R.metrics(kind, impl, s, n)
                    assert O.traffic(p, n) == R.traffic(kind, impl, s, n)
                finally:
                    O.free(p)
            for n in (3, 5):
                s = int(rng.integers(1, 5000))
                _, mine = O.run(kind, impl, s, n, seed=9)
                ref = R.execute(kind, impl, s, n, seed=9)
                assert all(np.array_equal(a, b) for a, b in zip(mine, ref))
