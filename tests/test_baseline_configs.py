"""GPU parity at the exact BASELINE.json configurations (SURVEY.md §8 sizing),
every byte of every rank's output against the reference's own digests
(tests/golden/baseline_configs.json, made by `python oracle/make_golden.py
baseline` from the reference's compile() + byte executor):

* C0 — all-gather, 8 ranks x 1 MiB (seeds 0 and 1);
* C1 — all-to-all, 8 ranks x 64 MiB send (s = 8 MiB), the bench headline;
* C4 — all-gather, 8 ranks x 256 MiB shards (2 GiB recv per rank).

The reference's six implementations are checked against their own digests;
the B200 executors (sm, hybrid, pull) against pcpy's — every implementation
has the same postcondition (verifier.cpp:143-169).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2511_06605_b200 as cc
from oracle import oracle as ora

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLDEN, "baseline_configs.json")) as _f:
    CASES = json.load(_f)

B200_EXTRA = ["sm", "hybrid", "pull"]


def _digest(cfg, impl, seed):
    ref_impl = impl if impl not in B200_EXTRA else "pcpy"
    for c in CASES:
        if (c["config"], c["impl"], c["seed"]) == (cfg, ref_impl, seed):
            return c
    raise KeyError((cfg, impl, seed))


def test_golden_file_covers_every_reference_implementation():
    for cfg, kind in (("C0", "allgather"), ("C1", "alltoall"), ("C4", "allgather")):
        impls = {c["impl"] for c in CASES if c["config"] == cfg}
        assert impls == set(ora.IMPLS_FOR[kind]), cfg
        # every implementation of the reference yields the same bytes
        assert len({tuple(c["sha256"]) for c in CASES if c["config"] == cfg and c["seed"] == 0}) == 1, cfg


def test_c0_digest_is_the_allgather_postcondition():
    """The golden all-gather output (verifier.cpp:143-169: out_g[k] = rank k's
    chunk for every g) restated from the inputs alone."""
    c = _digest("C0", "pcpy", 0)
    ins = [ora.splitmix_pattern(c["s"], r, 0) for r in range(c["n"])]
    want = hashlib.sha256(np.concatenate(ins).tobytes()).hexdigest()
    assert c["sha256"] == [want] * c["n"]


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------

_HOST = {}


def _inputs(kind, n, s, seed):
    key = (kind, n, s, seed)
    if key not in _HOST:
        _HOST.clear()
        in_bytes = s if kind == "allgather" else n * s
        _HOST[key] = [ora.splitmix_pattern(in_bytes, r, seed) for r in range(n)]
    return _HOST[key]


_COMMS = {}


def _comms(n):
    if n not in _COMMS:
        _COMMS[n] = cc.Comm.init_all([0] * n)
    return _COMMS[n]


def _run(torch, kind, impl, n, s, seed, per_rank):
    host = _inputs(kind, n, s, seed)
    sends = [torch.from_numpy(h).cuda() for h in host]
    in_place = impl.endswith("swap")
    recvs = sends if in_place else [torch.full((n * s,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(n)]
    streams = [torch.cuda.Stream() for _ in range(n)] if per_rank else torch.cuda.current_stream()
    if per_rank:
        for st in streams:
            st.wait_stream(torch.cuda.current_stream())
    torch.cuda.synchronize()
    fn = cc.all_gather if kind == "allgather" else cc.all_to_all
    # twice: the plan's first (eager) launch and its recorded replay
    for _ in range(2):
        if in_place:
            for t, h in zip(sends, host):
                t.copy_(torch.from_numpy(h))
            torch.cuda.synchronize()
        fn(_comms(n), sends, recvs, s, impl=impl, streams=streams)
        torch.cuda.synchronize()
    return recvs


def _sha_dev(t):
    return hashlib.sha256(memoryview(t.cpu().numpy())).hexdigest()


C0_IMPLS = ora.IMPLS_FOR["allgather"] + B200_EXTRA
C1_IMPLS = ora.IMPLS_FOR["alltoall"] + B200_EXTRA


@pytest.mark.gpu
@pytest.mark.parametrize("per_rank", [False, True], ids=["one_stream", "stream_per_rank"])
@pytest.mark.parametrize("seed", [0, 1])
@pytest.mark.parametrize("impl", C0_IMPLS)
def test_c0_allgather_8x1MiB(impl, seed, per_rank):
    torch = pytest.importorskip("torch")
    c = _digest("C0", impl, seed)
    recvs = _run(torch, "allgather", impl, c["n"], c["s"], seed, per_rank)
    assert [_sha_dev(r) for r in recvs] == c["sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("impl", C1_IMPLS)
def test_c1_alltoall_8x64MiB(impl):
    torch = pytest.importorskip("torch")
    c = _digest("C1", impl, 0)
    recvs = _run(torch, "alltoall", impl, c["n"], c["s"], 0, False)
    assert [_sha_dev(r) for r in recvs] == c["sha256"]


@pytest.mark.gpu
@pytest.mark.timeout(600)
@pytest.mark.parametrize("impl", C0_IMPLS)
def test_c4_allgather_8x256MiB(impl):
    """2 GiB per rank: every rank's recv must equal rank 0's byte for byte
    (compared on the device), and rank 0's digest must be the reference's."""
    torch = pytest.importorskip("torch")
    c = _digest("C4", impl, 0)
    assert len(set(c["sha256"])) == 1
    recvs = _run(torch, "allgather", impl, c["n"], c["s"], 0, False)
    for r in recvs[1:]:
        assert torch.equal(r, recvs[0])
    assert _sha_dev(recvs[0]) == c["sha256"][0]
    del recvs
    torch.cuda.empty_cache()
