"""Repeats the back-to-back stress of tests/test_gpu_parity.py many times and
classifies every mismatch (which iteration's bytes landed where): a
diagnostic for flag-protocol races. Usage:
  python tools/b2b_stress.py IMPL REPS [force|plain] [allgather|alltoall]"""
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 3 and sys.argv[3] == "force":
    os.environ["CECOLL_FORCE_REMOTE_SIGNALS"] = "1"
import numpy as np
import torch

import paper_2511_06605_b200 as cc
from oracle import oracle as ora


KIND = sys.argv[4] if len(sys.argv) > 4 else "alltoall"


def expected_alltoall(hosts_it, n, s):
    if KIND == "allgather":
        full = np.concatenate([hosts_it[j][:s] for j in range(n)])
        return [full for _ in range(n)]
    return [np.concatenate([hosts_it[j][r * s:(r + 1) * s] for j in range(n)]) for r in range(n)]


def one(impl, rep, n=4, s=12288 + 16, iters=12, fresh=True):
    cs = cc.Comm.init_all([0] * n)
    rng = random.Random(f"b2b-{impl}-{rep}")
    in_place = impl.endswith("swap")
    streams = [torch.cuda.Stream() for _ in range(n)]
    in_bytes = s if KIND == "allgather" else n * s
    hosts = [[ora.splitmix_pattern(in_bytes, r, 5000 + it) for r in range(n)] for it in range(iters)]
    inputs = [[torch.from_numpy(hosts[it][r]).cuda() for r in range(n)] for it in range(iters)]
    sends = [torch.empty(in_bytes, dtype=torch.uint8, device="cuda") for _ in range(n)]
    recvs = sends if in_place else [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
    outs = [[torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)] for _ in range(iters)]
    torch.cuda.synchronize()
    for it in range(iters):
        for r, st in enumerate(streams):
            with torch.cuda.stream(st):
                if rng.random() < 0.5:
                    torch.cuda._sleep(rng.randint(1000, 100000))
                sends[r].copy_(inputs[it][r])
        fn = cc.all_gather if KIND == "allgather" else cc.all_to_all
        fn(cs, sends, recvs, s, impl=impl, streams=streams)
        for r, st in enumerate(streams):
            with torch.cuda.stream(st):
                if rng.random() < 0.5:
                    torch.cuda._sleep(rng.randint(1000, 100000))
                outs[it][r].copy_(recvs[r])
    torch.cuda.synchronize()
    bad = []
    exps = [expected_alltoall(hosts[it], n, s) for it in range(iters)]
    for it in range(iters):
        for r in range(n):
            got = outs[it][r].cpu().numpy()
            if np.array_equal(got, exps[it][r]):
                continue
            for j in range(n):
                blk = got[j * s:(j + 1) * s]
                if np.array_equal(blk, exps[it][r][j * s:(j + 1) * s]):
                    continue
                where = [k for k in range(iters) if np.array_equal(blk, exps[k][r][j * s:(j + 1) * s])]
                nbad = int((blk != exps[it][r][j * s:(j + 1) * s]).sum())
                first = int(np.argmax(blk != exps[it][r][j * s:(j + 1) * s]))
                bad.append(dict(it=it, dst=r, src=j, nbad=nbad, first=first, matches_iter=where))
    cc.destroy_all(cs)
    return bad


if __name__ == "__main__":
    impl, reps = sys.argv[1], int(sys.argv[2])
    import time
    fails = 0
    for rep in range(reps):
        t0 = time.time()
        err = None
        try:
            b = one(impl, rep)
        except Exception as e:  # a timeout reported at destroy
            b, err = [], repr(e)
        dt = time.time() - t0
        if b or err or dt > 5:
            fails += 1
            print(f"rep {rep} ({dt:.1f} s) err={err}: {len(b)} bad blocks: {b[:4]}", flush=True)
    print(f"{KIND} {impl} force={os.environ.get('CECOLL_FORCE_REMOTE_SIGNALS', '0')}: {fails}/{reps} reps failed",
          flush=True)
