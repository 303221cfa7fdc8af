"""Reduce-scatter: the oracle against an independent numpy
restatement (CPU), and every implementation on the GPU bit-exact against the
oracle (fp32 accumulation in rank order, one round-to-nearest-even)."""
import numpy as np
import pytest

from oracle import oracle as ora

DT = {"f32": 0, "bf16": 1, "f16": 2}
OPS = {"sum": 0, "max": 1, "min": 2}


def _inputs(dtype, n, count, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, n * count)).astype(np.float32) * 4
    if dtype == "f32":
        return [r.view(np.uint8).copy() for r in x]
    if dtype == "f16":
        return [r.astype(np.float16).view(np.uint8).copy() for r in x]
    u = x.view(np.uint32)
    b = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)  # RNE to bf16
    return [r.view(np.uint8).copy() for r in b]


def _to_f32(buf, dtype):
    if dtype == "f32":
        return buf.view(np.float32)
    if dtype == "f16":
        return buf.view(np.float16).astype(np.float32)
    return (buf.view(np.uint16).astype(np.uint32) << 16).view(np.float32)


def _from_f32(x, dtype):
    if dtype == "f32":
        return x.astype(np.float32).view(np.uint8)
    if dtype == "f16":
        return x.astype(np.float16).view(np.uint8)
    u = x.astype(np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16).view(np.uint8)


def numpy_rs(ins, dtype, op, count):
    n = len(ins)
    xs = [_to_f32(b, dtype).reshape(n, count) for b in ins]
    outs = []
    for j in range(n):
        acc = xs[0][j].copy()
        for i in range(1, n):
            v = xs[i][j]
            if op == "sum":
                acc = (acc + v).astype(np.float32)
            elif op == "max":
                acc = np.where(v > acc, v, acc)
            else:
                acc = np.where(v < acc, v, acc)
        outs.append(_from_f32(acc, dtype))
    return outs


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
@pytest.mark.parametrize("op", ["sum", "max", "min"])
@pytest.mark.parametrize("n,count", [(2, 1000), (3, 4096), (8, 777)])
def test_oracle_matches_numpy(dtype, op, n, count):
    ins = _inputs(dtype, n, count, seed=n * count)
    got = ora.Oracle().reduce_scatter(DT[dtype], OPS[op], count, ins)
    want = numpy_rs(ins, dtype, op, count)
    assert all(np.array_equal(g, w) for g, w in zip(got, want))


@pytest.mark.gpu
@pytest.mark.parametrize("impl", ["sm", "pcpy", "b2b", "prelaunch_pcpy", "prelaunch_b2b"])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
@pytest.mark.parametrize("op", ["sum", "max"])
@pytest.mark.parametrize("n,count,streams", [(2, 4096, "shared"), (4, 1000, "per_rank"), (8, 65536 + 24, "shared"),
                                             (8, 262144 + 8, "per_rank")])
def test_gpu_matches_oracle(impl, dtype, op, n, count, streams):
    torch = pytest.importorskip("torch")
    import paper_2511_06605_b200 as cc

    comms = _comms(n)
    ins = _inputs(dtype, n, count, seed=7 + n)
    want = ora.Oracle().reduce_scatter(DT[dtype], OPS[op], count, ins)
    es = 4 if dtype == "f32" else 2
    sends = [torch.from_numpy(b).cuda() for b in ins]
    recvs = [torch.full((count * es,), 0xA5, dtype=torch.uint8, device="cuda") for _ in range(n)]
    sts = torch.cuda.current_stream() if streams == "shared" else [torch.cuda.Stream() for _ in range(n)]
    torch.cuda.synchronize()
    for _ in range(2):  # twice: plan reuse and flag resets
        cc.reduce_scatter(comms, sends, recvs, count, dtype=dtype, op=op, impl=impl, streams=sts)
    torch.cuda.synchronize()
    got = [r.cpu().numpy() for r in recvs]
    assert all(np.array_equal(g, w) for g, w in zip(got, want))


_C = {}


def _comms(n):
    import paper_2511_06605_b200 as cc

    if n not in _C:
        _C[n] = cc.Comm.init_all([0] * n)
    return _C[n]


@pytest.mark.gpu
@pytest.mark.timeout(300)
@pytest.mark.parametrize("impl,force_remote", [("sm", False), ("sm", True), ("pcpy", False), ("pcpy", True),
                                               ("b2b", False), ("prelaunch_pcpy", False), ("prelaunch_pcpy", True)])
def test_back_to_back_without_host_sync(impl, force_remote, monkeypatch):
    """The reader-side protocol of reduce-scatter (a reader waits for the
    owner's rdy and signals done back) under reuse: one stream per rank, per
    iteration a random spin, the input reload, the collective, a random spin
    and the copy-out, no host synchronisation. A send reloaded while a peer
    still reads it, or a result read before every chunk was folded, changes
    some iteration's bytes."""
    import random

    torch = pytest.importorskip("torch")
    import paper_2511_06605_b200 as cc

    if force_remote:
        monkeypatch.setenv("CECOLL_FORCE_REMOTE_SIGNALS", "1")
    n, count, iters = 4, 6144 + 8, 10
    comms = cc.Comm.init_all([0] * n)
    O = ora.Oracle()
    rng = random.Random(f"rs-{impl}-{force_remote}")
    ins = [_inputs("bf16", n, count, seed=500 + it) for it in range(iters)]
    wants = [O.reduce_scatter(DT["bf16"], OPS["sum"], count, ins[it]) for it in range(iters)]
    inputs = [[torch.from_numpy(b).cuda() for b in ins[it]] for it in range(iters)]
    sends = [torch.empty(n * count * 2, dtype=torch.uint8, device="cuda") for _ in range(n)]
    recvs = [torch.empty(count * 2, dtype=torch.uint8, device="cuda") for _ in range(n)]
    outs = [[torch.empty(count * 2, dtype=torch.uint8, device="cuda") for _ in range(n)] for _ in range(iters)]
    streams = [torch.cuda.Stream() for _ in range(n)]
    torch.cuda.synchronize()
    for it in range(iters):
        for r, st in enumerate(streams):
            with torch.cuda.stream(st):
                if rng.random() < 0.5:
                    torch.cuda._sleep(rng.randint(1000, 100000))
                sends[r].copy_(inputs[it][r])
        cc.reduce_scatter(comms, sends, recvs, count, dtype="bf16", op="sum", impl=impl, streams=streams)
        for r, st in enumerate(streams):
            with torch.cuda.stream(st):
                if rng.random() < 0.5:
                    torch.cuda._sleep(rng.randint(1000, 100000))
                outs[it][r].copy_(recvs[r])
    torch.cuda.synchronize()
    bad = [(it, r) for it in range(iters) for r in range(n)
           if not np.array_equal(outs[it][r].cpu().numpy(), wants[it][r])]
    assert comms[0].async_error() is None
    cc.destroy_all(comms)
    assert not bad, bad

