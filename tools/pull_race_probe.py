"""Two processes on one GPU, 2 ranks each, back-to-back all-to-alls without
host synchronisation (tests/test_multiprocess.py's stress worker), with a
diagnosis of every wrong chunk: which iteration's input of which source it
holds, if any.

  python tools/pull_race_probe.py [impls=swap,pull] [iters=40] [rounds=3] [force_remote=0]
"""
import os
import socket
import sys
import traceback

import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, port, impls, iters, rounds, force_remote, out):
    try:
        sys.path.insert(0, ROOT)
        if force_remote:
            os.environ["CECOLL_FORCE_REMOTE_SIGNALS"] = "1"
        import random

        import numpy as np
        import torch
        import torch.distributed as dist

        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
        import paper_2511_06605_b200 as cc
        from oracle import oracle as ora

        nranks, nlocal = 4, 2
        first = rank * nlocal
        comms = cc.Comm.init_ranks(nranks, first, nlocal, 0, cc.torch_exchange())
        s = 24576 + 32
        streams = [torch.cuda.Stream() for _ in range(nlocal)]
        wins = [torch.zeros(2 * nranks * s, dtype=torch.uint8, device="cuda") for _ in comms]
        for c, w in zip(comms, wins):
            c.register(w)
        report = []
        for rnd in range(rounds):
            for impl in impls:
                rng = random.Random(f"{impl}-{rank}-{rnd}")
                in_place = impl.endswith("swap")
                hosts = [[ora.splitmix_pattern(nranks * s, r, 9000 + 100 * rnd + it) for r in range(nranks)]
                         for it in range(iters)]
                inputs = [[torch.from_numpy(hosts[it][first + k]).cuda() for k in range(nlocal)] for it in range(iters)]
                outs = [[torch.empty(nranks * s, dtype=torch.uint8, device="cuda") for _ in range(nlocal)]
                        for _ in range(iters)]
                sends = [w[:nranks * s] for w in wins]
                recvs = sends if in_place else [w[nranks * s:] for w in wins]
                torch.cuda.synchronize()
                dist.barrier()
                for it in range(iters):
                    for k, st in enumerate(streams):
                        with torch.cuda.stream(st):
                            if rng.random() < 0.5:
                                torch.cuda._sleep(rng.randint(1000, 100000))
                            sends[k].copy_(inputs[it][k])
                    cc.all_to_all(comms, sends, recvs, s, impl=impl, streams=streams)
                    for k, st in enumerate(streams):
                        with torch.cuda.stream(st):
                            if rng.random() < 0.5:
                                torch.cuda._sleep(rng.randint(1000, 100000))
                            outs[it][k].copy_(recvs[k])
                torch.cuda.synchronize()
                nbad = 0
                for it in range(iters):
                    for k in range(nlocal):
                        r = first + k
                        got = outs[it][k].cpu().numpy()
                        for j in range(nranks):
                            want = hosts[it][j][r * s:(r + 1) * s]
                            g = got[j * s:(j + 1) * s]
                            if np.array_equal(g, want):
                                continue
                            nbad += 1
                            what = "unknown"
                            for it2 in range(iters):
                                if np.array_equal(g, hosts[it2][j][r * s:(r + 1) * s]):
                                    what = f"input of iteration {it2}"
                                    break
                            frac = float(np.mean(g != want))
                            report.append(f"round {rnd} {impl} it {it} rank {r} slot {j} (source {j}"
                                          f"{' local' if j // nlocal == rank else ' other process'}): "
                                          f"{frac:.3f} of bytes differ; holds {what}")
                report.append(f"round {rnd} {impl}: {nbad} bad chunks of {iters * nlocal * nranks}")
                dist.barrier()
        err = comms[0].async_error()
        report.append(f"async_error {err}")
        out.put((rank, report))
        torch.cuda.synchronize()
        for c in comms:
            c.destroy()
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        out.put((rank, [traceback.format_exc()]))


if __name__ == "__main__":
    impls = (sys.argv[1] if len(sys.argv) > 1 else "swap,pull").split(",")
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    force_remote = len(sys.argv) > 4 and sys.argv[4] == "1"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=worker, args=(r, port, impls, iters, rounds, force_remote, q)) for r in range(2)]
    for p in procs:
        p.start()
    for _ in procs:
        rank, rep = q.get(timeout=900)
        for line in rep:
            print(f"[proc {rank}] {line}", flush=True)
    for p in procs:
        p.join(timeout=60)
