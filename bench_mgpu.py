"""Multi-GPU arm of bench.py: torchrun, one process per GPU (N = 2, 4, 8).

Only the driver's round-end scaling run executes this across GPUs (in-round
GPU calls get one GPU; there the same code runs with N processes sharing
cuda:0, NCCL skipped), so it is written to finish with a JSON line whatever
happens:

* every implementation is tried under cross-rank consensus — a plan that
  fails to build, raises, or breaks parity on any rank is dropped on every
  rank before anything waits on its flags — and the fastest parity-clean one
  is the headline (the run-time analogue of winner_grid, sweep.cpp:186-218);
* a watchdog prints what was measured so far and exits if a collective
  never completes.

Headline (BASELINE.json configs[1], strong scaling): the 8-rank all-to-all of
8 x 64 MiB with 8/N ranks co-resident per GPU, device-timed, max over ranks.
Beside it, in the same run: NCCL (torch.distributed, backend nccl) moving the
same cross-GPU bytes, e2e through the plans with pinned host buffers, and a
4 KiB-1 GiB all-gather / all-to-all sweep with one rank per GPU (n = N)
against NCCL (BASELINE.json configs[2], [3]).
"""
from __future__ import annotations

import datetime
import json
import os
import threading
import time

import torch
import torch.distributed as dist

import paper_2511_06605_b200 as cc

NVLINK_PEAK = 770.0  # measured peer copy GB/s per direction (B200_PROFILING.md)
NVLINK_NOMINAL = 900.0

# Per sweep size, the prelaunch forms last: their cross-device bodies are
# conditional graphs with copy-engine nodes, the least exercised form.
AG_IMPLS = ["sm", "pcpy", "b2b", "bcst", "hybrid", "pull", "prelaunch_pcpy", "prelaunch_b2b", "prelaunch_bcst"]
AA_IMPLS = ["sm", "pcpy", "b2b", "swap", "hybrid", "pull", "prelaunch_pcpy", "prelaunch_b2b", "prelaunch_swap"]
# Headline trials: every non-prelaunch form plus the hybrid's SM-share scan
# ("impl@pct": CECOLL_HYBRID_SM_PCT at plan creation). The prelaunch forms
# are measured in the sweep, after the headline is in the line.
HEADLINE_IMPLS = ["sm", "pcpy", "b2b", "swap", "hybrid", "pull", "hybrid@25", "hybrid@75"]

STATE: dict = {}  # what the watchdog prints if a collective hangs
ASYNC_NOTES: list = []  # device-side poll timeouts reported when a phase's world is destroyed


def quiet_destroy(objs):
    """Destroy communicators without raising: a device-side poll timeout that
    a phase's world recorded (cecoll_comm_destroy's async error) is noted in
    the line (`async_errors`) instead of ending the run before it prints."""
    for o in objs:
        try:
            o.destroy()
        except cc.CecollError as e:
            ASYNC_NOTES.append(f"{STATE.get('phase', '?')}: {str(e)[:200]}")


# ---------------------------------------------------------------------------
# cross-rank helpers (gloo, CPU tensors)
# ---------------------------------------------------------------------------


def all_true(flag: bool) -> bool:
    t = torch.tensor([1 if flag else 0], dtype=torch.int32)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def max_all(x: float) -> float:
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def from_rank0(x):
    box = [x]
    dist.broadcast_object_list(box, src=0)
    return box[0]


class Watchdog:
    def __init__(self, seconds: float, rank: int, line_fn):
        self.rank, self.line_fn = rank, line_fn
        self.t = threading.Timer(seconds, self._fire)
        self.t.daemon = True
        self.t.start()

    def _fire(self):
        phase = str(STATE.get("phase"))
        in_experiments = phase.startswith("experiment")
        try:  # every rank holds the same line (value set on all ranks)
            headline_done = self.line_fn().get("value") is not None
        except Exception:  # noqa: BLE001
            headline_done = False
        if self.rank == 0:
            try:
                line = self.line_fn()
                if in_experiments:  # the main measurement is complete
                    line.setdefault("experiments", {})["hung"] = phase
                else:
                    line["error"] = f"watchdog: a collective did not complete (phase {phase})"
                trials = {k: v for k, v in line["details"].get("impl_trials", {}).items() if "ms" in v}
                if line.get("value") is None and trials:
                    best = min(trials, key=lambda k: trials[k]["ms"])
                    line["value"] = trials[best]["busbw_gbs"]
                    line["ms_per_step"] = trials[best]["ms"]
                    line["details"]["impl"] = best + " (from the trial phase)"
                print(json.dumps(line), flush=True)
            except Exception:  # noqa: BLE001
                pass
        # The headline (value) was measured before the hang: the run stands,
        # with the hung phase named in the line.
        os._exit(0 if in_experiments or headline_done else 1)

    def cancel(self):
        self.t.cancel()


# ---------------------------------------------------------------------------
# synthetic chunks: chunk (src rank i -> dst rank j) is a seeded byte pattern,
# so any process can rebuild what it must receive without the sender's data
# ---------------------------------------------------------------------------


def pattern(seed: int, nbytes: int, dev) -> torch.Tensor:
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    return torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=dev, generator=g)


def seed_of(kind: str, s: int, i: int, j: int) -> int:
    k = 0 if kind == "allgather" else 1
    return ((s.bit_length() * 64 + i) * 64 + (0 if kind == "allgather" else j)) * 2 + k


def fill_and_expect(kind, s, n, ranks, sends, expects, dev):
    """sends[k] of global rank ranks[k]; expects[k] is what that rank must receive."""
    for r, snd in zip(ranks, sends):
        if kind == "allgather":
            snd[:s].copy_(pattern(seed_of(kind, s, r, 0), s, dev))
        else:
            for j in range(n):
                snd[j * s:(j + 1) * s].copy_(pattern(seed_of(kind, s, r, j), s, dev))
    for r, exp in zip(ranks, expects):
        for i in range(n):
            exp[i * s:(i + 1) * s].copy_(pattern(seed_of(kind, s, i, r), s, dev))


# ---------------------------------------------------------------------------
# one implementation: build (consensus), parity (consensus), timing (max)
# ---------------------------------------------------------------------------


def make_plan(comms, kind, sends, recvs, s, impl):
    """cc.Plan for an implementation name, or "name@pct" for the hybrid's SM
    share (CECOLL_HYBRID_SM_PCT, read at plan creation)."""
    name, _, pct = impl.partition("@")
    saved = os.environ.get("CECOLL_HYBRID_SM_PCT")
    if pct:
        os.environ["CECOLL_HYBRID_SM_PCT"] = pct
    try:
        return cc.Plan(comms, kind, sends, recvs, s, impl=name)
    finally:
        if pct:
            if saved is None:
                os.environ.pop("CECOLL_HYBRID_SM_PCT", None)
            else:
                os.environ["CECOLL_HYBRID_SM_PCT"] = saved


def try_impl(comms, kind, impl, sends, recvs, expects, s, iters, stream):
    """Returns (plan or None, result dict). The plan is left disarmed."""
    in_place = impl.endswith("swap")
    for r, snd in zip(recvs, sends):
        if in_place:
            r.copy_(snd)
        else:
            r.fill_(0xA5)
    torch.cuda.synchronize()
    plan, err = None, None
    try:
        plan = make_plan(comms, kind, recvs if in_place else sends, recvs, s, impl)
    except cc.CecollError as e:
        err = str(e)[:160]
    if not all_true(plan is not None):
        if plan is not None:
            plan.destroy()
        return None, {"error": err or "plan failed on another rank"}
    dist.barrier()
    STATE["phase"] = f"{STATE.get('prefix', '')}{kind} {impl} s={s} parity"
    try:
        plan.launch(stream)
        stream.synchronize()
        plan.disarm()
        ok = all(bool(torch.equal(r, e)) for r, e in zip(recvs, expects))
    except cc.CecollError as e:
        ok, err = False, str(e)[:160]
    if not all_true(ok):
        try:
            plan.disarm()
            torch.cuda.synchronize()
            plan.destroy()
        except cc.CecollError:
            pass
        return None, {"error": err or "parity failed"}
    STATE["phase"] = f"{STATE.get('prefix', '')}{kind} {impl} s={s} timing"
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        plan.launch(stream)
    stream.synchronize()
    dist.barrier()
    e0.record(stream)
    for _ in range(iters):
        plan.launch(stream)
    e1.record(stream)
    stream.synchronize()
    plan.disarm()
    ms = max_all(e0.elapsed_time(e1) / iters)
    return plan, {"ms": ms, "plan": plan_summary(plan)}


def plan_summary(plan):
    """cecoll_plan_info reduced to what a reader needs to trust the number:
    graph fallback, recording, mover per unit, how flags between units travel."""
    try:
        i = plan.info()
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)[:120]}
    return {"graph_fallback": i.get("graph_fallback", ""), "recorded": i.get("recorded"),
            "record_note": i.get("record_note", ""), "prelaunch_folded": i.get("prelaunch_folded"),
            "remote_signals": i.get("remote_signals"), "sm_budget": i.get("sm_budget"),
            "movers": [u.get("mover") for u in i.get("units", [])],
            "ce_lanes": [u.get("ce_lanes") for u in i.get("units", [])],
            "fused_flags": [u.get("fused_flags") for u in i.get("units", [])],
            "flag_writes_kernel": [u.get("flag_writes_kernel") for u in i.get("units", [])],
            "flag_writes_memop": [u.get("flag_writes_memop") for u in i.get("units", [])]}


def energy_loop(step, stream, dev, n, s, plan, seconds=1.5):
    """J/GB over a loop of `step` on every GPU: the collective count is rank
    0's (all ranks run the same count), energy is summed over ranks."""
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(dev)
    except Exception as e:  # noqa: BLE001
        all_true(False)
        return {"error": f"nvml: {str(e)[:80]}"}
    if not all_true(True):
        return {"error": "nvml unavailable on a rank"}
    step()
    stream.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        step()
    stream.synchronize()
    per = max(1e-6, (time.perf_counter() - t0) / 20)
    count = int(from_rank0(int(max(40, seconds / per))))
    dist.barrier()
    e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
    t0 = time.perf_counter()
    for k in range(count):
        step()
        if k % 50 == 49:
            stream.synchronize()  # bounded queue
    stream.synchronize()
    dt = time.perf_counter() - t0
    e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
    if plan is not None:
        plan.disarm()
    t = torch.tensor([(e1 - e0) / 1e3, dt], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    joules, secs = float(t[0]), float(t[1]) / dist.get_world_size()
    gb = n * (n - 1) * s * count / 1e9
    return {"j_per_gb": round(joules / gb, 5), "joules": round(joules, 2), "seconds": round(secs, 3),
            "collectives": count, "avg_power_w_per_gpu": round(joules / secs / dist.get_world_size(), 1)}


def time_nccl(group, kind, send, recv, iters, stream):
    if group is None:
        return None
    STATE["phase"] = f"nccl {kind}"

    def op():
        if kind == "allgather":
            dist.all_gather_into_tensor(recv, send, group=group)
        else:
            dist.all_to_all_single(recv, send, group=group)

    with torch.cuda.stream(stream):
        for _ in range(3):
            op()
        stream.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            op()
        e1.record(stream)
    stream.synchronize()
    return max_all(e0.elapsed_time(e1) / iters)


def topology(dev: int, world: int) -> dict:
    """What the box offers beyond what one-GPU development boxes show: copy
    engines, switch multicast (NVLS; a probe cuMulticastCreate for N devices),
    peer access, active NVLink links. Reported for the next design round."""
    import ctypes as C

    out: dict = {"visible_gpus": torch.cuda.device_count()}
    try:
        cu = C.CDLL("libcuda.so.1")
        cu.cuInit(0)
        d = C.c_int()
        cu.cuDeviceGet(C.byref(d), dev)
        for name, attr in (("async_engine_count", 40), ("multicast_supported", 132)):
            v = C.c_int(-1)
            cu.cuDeviceGetAttribute(C.byref(v), attr, d)
            out[name] = v.value

        class McProp(C.Structure):
            _fields_ = [("numDevices", C.c_uint), ("size", C.c_size_t), ("handleTypes", C.c_ulonglong),
                        ("flags", C.c_ulonglong)]

        for ht, label in ((1, "posix_fd"), (8, "fabric")):
            prop = McProp(world, 2 << 20, ht, 0)
            h = C.c_ulonglong()
            r = cu.cuMulticastCreate(C.byref(h), C.byref(prop))
            out[f"multicast_create_{label}_n{world}"] = int(r)
            if r == 0:
                cu.cuMemRelease(h)
    except Exception as e:  # noqa: BLE001
        out["cuda_probe_error"] = str(e)[:120]
    try:
        out["peer_access"] = all(torch.cuda.can_device_access_peer(dev, o)
                                 for o in range(torch.cuda.device_count()) if o != dev)
    except Exception:  # noqa: BLE001
        pass
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(dev)
        active = 0
        for link in range(18):
            try:
                active += int(pynvml.nvmlDeviceGetNvLinkState(h, link) == 1)
            except Exception:  # noqa: BLE001
                break
        out["nvlink_active_links"] = active
        out["driver"] = pynvml.nvmlSystemGetDriverVersion()
    except Exception:  # noqa: BLE001
        pass
    return out


def busbw(n, s, ms):
    return (n - 1) * s / (ms / 1e3) / 1e9


# ---------------------------------------------------------------------------
# the run
# ---------------------------------------------------------------------------


def run(args, B):
    t_start = time.time()
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    n, s = B.NRANKS, B.CHUNK
    if n % world:
        raise SystemExit(f"--gpus must divide {n}")
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=900))
    nlocal = n // world
    first = rank * nlocal
    my_ranks = list(range(first, first + nlocal))

    line = {
        "metric": B.METRIC, "value": None, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded torch.randint byte chunks)",
        "config": B.bench_config(),
        "details": {"ranks_per_gpu": nlocal,
                    "l2": "inputs larger than L2 (64 MiB send + 64 MiB recv per rank)"},
    }
    dog = Watchdog(args.mgpu_deadline, rank, lambda: line)

    uuids = [None] * world
    dist.all_gather_object(uuids, str(torch.cuda.get_device_properties(dev).uuid))
    distinct = len(set(uuids)) == world
    nccl = None
    nccl_note = None
    if not distinct:
        nccl_note = "skipped: several processes share one GPU (NCCL rejects duplicate devices)"
    elif args.no_nccl:
        nccl_note = "skipped (--no-nccl)"
    else:
        try:
            nccl = dist.new_group(backend="nccl")
        except Exception as e:  # noqa: BLE001
            nccl_note = f"unavailable: {str(e)[:120]}"
    line["details"]["gpus_distinct"] = distinct
    if rank == 0:
        line["topology"] = topology(dev, world)

    stream = torch.cuda.Stream()
    STATE["phase"] = "init"
    # Communicator and two symmetric windows per rank, [send n*s | recv n*s]
    # (double-buffered e2e). Both are collective (exchange over gloo), so a
    # failure on one rank surfaces as an exchange failure on the others;
    # either way every rank reports and the line still carries NCCL.
    comms, sets, init_err = None, [], None
    try:
        comms = cc.Comm.init_ranks(n, first, nlocal, dev, cc.torch_exchange())
        for _b in range(2):
            wins = [torch.empty(2 * n * s, dtype=torch.uint8, device="cuda") for _ in comms]
            for c, w in zip(comms, wins):
                c.register(w)
            sets.append(([w[:n * s] for w in wins], [w[n * s:] for w in wins]))
    except Exception as e:  # noqa: BLE001
        init_err = str(e)[:200]
    if not all_true(init_err is None):
        line["error"] = f"communicator / window setup failed: {init_err or 'on another rank'}"
        if nccl is not None:
            inp = torch.empty(nlocal * n * s, dtype=torch.uint8, device="cuda")
            t = time_nccl(nccl, "alltoall", inp, torch.empty_like(inp), args.steps, stream)
            line["nccl"] = {"value": round(busbw(n, s, t), 3), "unit": "GB/s", "ms_per_step": round(t, 4)}
        if rank == 0:
            print(json.dumps(line), flush=True)
        dog.cancel()
        return
    sends, recvs = sets[0]
    expects = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in comms]
    fill_and_expect("alltoall", s, n, my_ranks, sends, expects, "cuda")
    torch.cuda.synchronize()

    # --- implementation trials (consensus), then the winner -----------------
    cands = HEADLINE_IMPLS if args.algo == "auto" else [args.algo]
    trials, plans = {}, {}
    line["details"]["impl_trials"] = trials
    for impl in cands:
        plan, res = try_impl(comms, "alltoall", impl, sends, recvs, expects, s, 10, stream)
        if plan is not None:
            plans[impl] = plan
            res["busbw_gbs"] = round(busbw(n, s, res["ms"]), 2)
            res["ms"] = round(res["ms"], 4)
        trials[impl] = res
    line["details"]["impl_trials"] = trials
    if not plans:
        line["error"] = "no implementation passed parity on every rank"
        if rank == 0:
            print(json.dumps(line), flush=True)
        dog.cancel()
        return
    best = min(plans, key=lambda k: trials[k]["ms"])
    best = from_rank0(best)
    line["details"]["impl"] = best
    plan = plans[best]
    line["details"]["plan"] = trials[best].get("plan")

    STATE["phase"] = "headline"
    if best.endswith("swap"):
        for r, snd in zip(recvs, sends):
            r.copy_(snd)
    for _ in range(max(3, args.warmup)):
        plan.launch(stream)
    stream.synchronize()
    plan.disarm()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with B.ClockSampler(dev) as clocks:
        torch.cuda.synchronize()
        dist.barrier()
        c0 = comms[0].counters()
        e0.record(stream)
        for _ in range(args.steps):
            plan.launch(stream)
        e1.record(stream)
        stream.synchronize()
        c1 = comms[0].counters()
        plan.disarm()
        torch.cuda.synchronize()
        dist.barrier()
    ms = max_all(e0.elapsed_time(e1) / args.steps)
    value = busbw(n, s, ms)
    if best.endswith("swap"):  # an even number of in-place transposes restores the input
        ok = True
    else:
        ok = all(bool(torch.equal(r, e)) for r, e in zip(recvs, expects))
    ok = all_true(ok)
    egress = nlocal * (n - nlocal) * s  # bytes leaving each GPU per collective
    nv = egress / (ms / 1e3) / 1e9
    # the bound for this N: NVLink egress, or the GPU's own HBM traffic
    # (every chunk of its ranks read once, every chunk for its ranks written once)
    hbm_peak = B.load_peaks()[0]
    bound_s = max(egress / (NVLINK_PEAK * 1e9), 2 * nlocal * n * s / (hbm_peak * 1e9))
    per = {k: (c1[k] - c0[k]) / args.steps for k in ("kernels", "graph_launches", "copies", "api_calls")}
    line.update({
        "value": round(value, 3), "ms_per_step": round(ms, 4), "parity_ok": ok,
        "roofline": {"bound": "nvlink", "achieved": round(nv, 1), "peak": NVLINK_PEAK, "unit": "GB/s",
                     "frac": round(nv / NVLINK_PEAK, 4), "traffic": None,
                     "frac_of_nominal_900": round(nv / NVLINK_NOMINAL, 4),
                     "peak_source": "measured peer copy per direction per GPU (B200_PROFILING.md)",
                     "algorithmic_bytes_per_gpu": egress,
                     "busbw_bound_gbs": round(busbw(n, s, bound_s * 1e3), 1),
                     "bound_note": "max(NVLink egress / 770 GB/s, local HBM traffic / measured copy peak)"},
        "gpu_launches": int(round((per["kernels"] + 4 * per["graph_launches"]) * args.steps)),
        "launches_note": "kernels + 4 per recorded-graph launch (gate, poll, items, signal) in the timed "
                         "region on rank 0; copy-engine copies are counted in config.ce_copies_per_step",
        "clocks": clocks.summary(),
    })
    line["details"]["ce_copies_per_step"] = per["copies"]
    line["details"]["api_calls_per_step"] = per["api_calls"]

    # --- NCCL moving the same cross-GPU bytes ----------------------------------
    if nccl is not None:
        inp = torch.empty(nlocal * n * s, dtype=torch.uint8, device="cuda")
        out = torch.empty_like(inp)
        t = time_nccl(nccl, "alltoall", inp, out, args.steps, stream)
        line["nccl"] = {"value": round(busbw(n, s, t), 3), "unit": "GB/s", "ms_per_step": round(t, 4),
                        "how": f"torch.distributed all_to_all_single of {nlocal * n * s >> 20} MiB per GPU "
                               f"(NCCL {'.'.join(map(str, torch.cuda.nccl.version()))}), same busBW convention",
                        "ours_over_nccl": round(t / ms, 3)}
        del inp, out
    else:
        line["nccl"] = {"value": None, "note": nccl_note}

    # --- NVML energy per link-equivalent GB, summed over the GPUs --------------
    STATE["phase"] = "energy"
    line["energy"] = {"ours": energy_loop(lambda: plan.launch(stream), stream, dev, n, s, plan)}
    if nccl is not None:
        inp = torch.empty(nlocal * n * s, dtype=torch.uint8, device="cuda")
        out = torch.empty_like(inp)

        def nccl_step():
            with torch.cuda.stream(stream):
                dist.all_to_all_single(out, inp, group=nccl)

        line["energy"]["nccl"] = energy_loop(nccl_step, stream, dev, n, s, None)
        del inp, out
    line["energy"]["note"] = ("NVML total energy of every GPU over a >= 1.5 s loop (rank 0 decides the "
                              "count), summed / link-equivalent bytes n(n-1)s per collective")

    # --- e2e: pinned host -> HBM -> collective -> HBM -> pinned host ----------
    STATE["phase"] = "e2e"
    line["e2e"] = run_e2e(comms, plans, best, sets, expects, s, n, nlocal, stream, args)

    for p in plans.values():
        p.destroy()
    plans.clear()
    torch.cuda.synchronize()
    dist.barrier()

    # --- sweep, one rank per GPU (n = N) ----------------------------------------
    if not args.no_mgpu_sweep:
        STATE["phase"] = "sweep"
        line["sweep"] = {"rows": []}
        line["sweep"] = run_sweep(world, rank, dev, nccl, stream, t_start, args, line["sweep"]["rows"])
    if not args.no_mgpu_interference and from_rank0(time.time() - t_start < args.mgpu_budget + 120):
        STATE["phase"] = "interference"
        line["interference"] = {}
        run_interference(world, rank, dev, nccl, stream, args, line["interference"])
    if not args.no_mgpu_interference and from_rank0(time.time() - t_start < args.mgpu_budget + 150):
        STATE["phase"] = "sync chain"
        line["sync_chain"] = {}
        run_sync_chain(world, rank, dev, stream, line["sync_chain"])
    if not args.no_mgpu_experiments:
        STATE["phase"] = "experiments"
        line["experiments"] = {}
        run_experiments(comms, sets, n, s, my_ranks, stream, line["experiments"])
    if not args.no_mgpu_sweep and "sweep" in line:
        STATE["phase"] = "experiments-grade sweep (prelaunch forms)"
        STATE["prefix"] = "experiments-grade sweep: "  # a hang here leaves the main line standing
        sweep_pass(world, rank, dev, nccl, stream, t_start, args, line["sweep"]["rows"], prelaunch=True)
        STATE["prefix"] = ""
    if not args.no_mgpu_experiments and from_rank0(time.time() - t_start < args.mgpu_budget + 220):
        STATE["phase"] = "experiments ce share"
        run_ce_share_experiment(world, rank, dev, line["experiments"])
    if not args.no_mgpu_experiments and from_rank0(time.time() - t_start < args.mgpu_budget + 240):
        STATE["phase"] = "experiments tune"
        run_tune_experiment(world, rank, dev, stream, line["experiments"])
    if not args.no_mgpu_experiments:
        STATE["phase"] = "experiments multicast"
        run_mc_experiment(world, rank, dev, stream, line["experiments"])
    line["details"]["wall_s"] = round(time.time() - t_start, 1)
    err = comms[0].async_error()
    if err is not None:
        ASYNC_NOTES.append(f"headline world: {str(err)[:200]}")
    if ASYNC_NOTES:
        line["async_errors"] = ASYNC_NOTES
    if rank == 0:
        print(json.dumps(line), flush=True)
    dog.cancel()
    torch.cuda.synchronize()
    dist.barrier()
    quiet_destroy(comms)
    dist.destroy_process_group()


def run_e2e(comms, plans, best, sets, expects, s, n, nlocal, stream, args):
    in_place = best.endswith("swap")
    e2e_plans = [plans[best]]
    try:
        s1, r1 = sets[1]
        e2e_plans.append(make_plan(comms, "alltoall", r1 if in_place else s1, r1, s, best))
    except cc.CecollError:
        e2e_plans = None
    if not all_true(e2e_plans is not None):
        return {"value": None, "error": "second plan failed"}
    sends0 = sets[0][0]
    host_in = [torch.empty(n * s, dtype=torch.uint8, pin_memory=True) for _ in comms]
    for h, d in zip(host_in, sends0):
        h.copy_(d)
    host_outs = [[torch.empty(n * s, dtype=torch.uint8, pin_memory=True) for _ in comms] for _ in range(2)]
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    in_ready = [torch.cuda.Event() for _ in range(2)]
    coll_done = [torch.cuda.Event() for _ in range(2)]
    out_done = [torch.cuda.Event() for _ in range(2)]
    for ev in coll_done + out_done:
        ev.record(stream)

    def step(k):
        b = k % 2
        sd, rv = sets[b]
        dst = rv if in_place else sd  # in place: the input lands in the in-place buffer
        h2d_s.wait_event(coll_done[b])
        h2d_s.wait_event(out_done[b])
        with torch.cuda.stream(h2d_s):
            for h, d in zip(host_in, dst):
                d.copy_(h, non_blocking=True)
        in_ready[b].record(h2d_s)
        stream.wait_event(in_ready[b])
        stream.wait_event(out_done[b])
        e2e_plans[b].launch(stream)
        coll_done[b].record(stream)
        d2h_s.wait_event(coll_done[b])
        with torch.cuda.stream(d2h_s):
            for h, d in zip(host_outs[b], rv):
                h.copy_(d, non_blocking=True)
        out_done[b].record(d2h_s)

    steps = max(getattr(args, "e2e_steps", 40), args.steps)
    for k in range(2):
        step(k)
    d2h_s.synchronize()
    stream.synchronize()
    for p in e2e_plans:
        p.disarm()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # cold window (pipeline empty at the start, drained at the end), then a
    # steady window (pipeline full at both edges) as in bench.py
    e0.record(h2d_s)
    k = 0
    for _ in range(steps):
        step(k)
        k += 1
    e1.record(d2h_s)
    for _ in range(2):
        step(k)
        k += 1
    s0.record(d2h_s)
    for _ in range(steps):
        step(k)
        k += 1
    s1.record(d2h_s)
    d2h_s.synchronize()
    stream.synchronize()
    for p in e2e_plans:
        p.disarm()
    torch.cuda.synchronize()
    cold = max_all(e0.elapsed_time(e1) / steps)
    ms = max_all(s0.elapsed_time(s1) / steps)
    last = host_outs[(k - 1) % 2]
    ok = all_true(all(bool(torch.equal(h.cuda(), e)) for h, e in zip(last, expects)))
    e2e_plans[1].destroy()
    return {"value": round(busbw(n, s, ms), 3), "unit": "GB/s", "h2d_bytes_per_step": n * n * s,
            "d2h_bytes_per_step": n * n * s, "ms_per_step": round(ms, 3), "parity_ok": ok, "steps": steps,
            "window": "steady state (pipeline full at both edges)", "cold_ms_per_step": round(cold, 3),
            "cold_value": round(busbw(n, s, cold), 3),
            "pipeline": "double-buffered: H2D of step k+1 overlaps D2H of step k; each GPU copies its "
                        f"{nlocal} ranks' buffers over its own PCIe link; bytes are whole-job"}


def summarize(row):
    """Winner and roofline fractions of one sweep row (recomputed whenever a
    pass adds implementations)."""
    ours = {k: v for k, v in row["us"].items() if v is not None and k != "nccl"}
    if not ours:
        return
    row["best"] = min(ours, key=ours.get)
    # fraction of the NVLink roofline (measured 770 GB/s per direction; busBW is per-GPU egress)
    row["best_frac_nvlink"] = round(row["busbw"][row["best"]] / NVLINK_PEAK, 4)
    if row["us"].get("nccl"):
        row["best_over_nccl_time"] = round(ours[row["best"]] / row["us"]["nccl"], 3)
        row["nccl_frac_nvlink"] = round(row["busbw"]["nccl"] / NVLINK_PEAK, 4)


def sweep_pass(world, rank, dev, nccl, stream, t_start, args, rows, prelaunch):
    """One pass over (kind, size): the non-prelaunch implementations with NCCL
    and the reduce-scatter (prelaunch=False, new rows), or only the prelaunch
    forms, merged into the existing rows (prelaunch=True, run near the end:
    their cross-device bodies are the least exercised graphs)."""
    n = world
    smax = 1 << int(args.mgpu_sweep_max).bit_length() - 1
    comms = cc.Comm.init_ranks(n, rank, 1, dev, cc.torch_exchange())
    win = torch.empty(2 * n * smax, dtype=torch.uint8, device="cuda")
    comms[0].register(win)
    exp = torch.empty(n * smax, dtype=torch.uint8, device="cuda")
    sizes = []
    s = 4096
    while s <= smax:
        sizes.append(s)
        s *= 4
    by_key = {(r["kind"], r["s"]): r for r in rows}
    for kind in ("allgather", "alltoall"):
        impls = [i for i in (AG_IMPLS if kind == "allgather" else AA_IMPLS) if i.startswith("prelaunch") == prelaunch]
        for s in sizes:
            row = by_key.get((kind, s))
            if prelaunch and (row is None or "skipped" in row):
                continue
            if not from_rank0(time.time() - t_start < (args.mgpu_budget if not prelaunch else args.mgpu_budget + 180)):
                if row is None:
                    rows.append({"kind": kind, "s": s, "skipped": "time budget"})
                continue
            if row is None:
                row = {"kind": kind, "s": s, "us": {}, "busbw": {}}
                rows.append(row)
            in_bytes = s if kind == "allgather" else n * s
            send = win[:in_bytes]
            recv = win[n * smax:n * smax + n * s]
            e = exp[:n * s]
            fill_and_expect(kind, s, n, [rank], [send], [e], "cuda")
            torch.cuda.synchronize()
            iters = int(max(5, min(100, 4e8 / max(1, (n - 1) * s))))
            for impl in impls:
                if impl.endswith("swap") and n < 2:
                    continue
                plan, res = try_impl(comms, kind, impl, [send], [recv], [e], s, iters, stream)
                if plan is None:
                    row["us"][impl] = None
                    row.setdefault("errors", {})[impl] = res.get("error")
                    continue
                plan.destroy()
                row["us"][impl] = round(res["ms"] * 1e3, 2)
                row["busbw"][impl] = round(busbw(n, s, res["ms"]), 2)
            if nccl is not None and not prelaunch:
                t = time_nccl(nccl, kind, send, recv, iters, stream)
                row["us"]["nccl"] = round(t * 1e3, 2)
                row["busbw"]["nccl"] = round(busbw(n, s, t), 2)
            summarize(row)
            if rank == 0 and args.mgpu_verbose:
                print(json.dumps(row), flush=True)
    if not prelaunch:
        # reduce-scatter, bf16 sum: the SM path (every rank
        # reads its chunk from every peer over NVLink) against NCCL.
        for s in [x for x in (65536, 1 << 20, 16 << 20, 256 << 20) if x <= smax]:
            if not from_rank0(time.time() - t_start < args.mgpu_budget):
                rows.append({"kind": "reduce_scatter_bf16_sum", "s": s, "skipped": "time budget"})
                continue
            row = {"kind": "reduce_scatter_bf16_sum", "s": s, "us": {}, "busbw": {}}
            rows.append(row)
            count = s // 2
            send, recv = win[:n * s], win[n * smax:n * smax + s]
            row.update(rs_trial(comms, nccl, send, recv, count, n, rank, stream))
            if rank == 0 and args.mgpu_verbose:
                print(json.dumps(row), flush=True)
    torch.cuda.synchronize()
    dist.barrier()
    quiet_destroy(comms[:1])
    del win, exp


def run_sweep(world, rank, dev, nccl, stream, t_start, args, rows):
    """AG and AA with one rank per GPU: every non-prelaunch implementation
    (consensus, parity) and NCCL per size, then the reduce-scatter; latency in
    us and busBW in GB/s. The prelaunch forms are added by a later pass."""
    sweep_pass(world, rank, dev, nccl, stream, t_start, args, rows, prelaunch=False)
    return {"ranks": world, "ranks_per_gpu": 1, "convention": "us = device time per collective (back to back, "
            "max over ranks); busbw = (n-1)*s/t; prelaunch forms added late in the run", "rows": rows}


def bf16_chunk(i: int, j: int, count: int) -> torch.Tensor:
    g = torch.Generator(device="cuda")
    g.manual_seed(((count.bit_length() * 64 + i) * 64 + j) * 2 + 7)
    return torch.randn(count, generator=g, device="cuda").to(torch.bfloat16)


def rs_trial(comms, nccl, send, recv, count, n, rank, stream):
    """Reduce-scatter, bf16 sum: chunk (i -> j) is seeded, so every rank
    rebuilds its expected result — the fp32 fold over ranks in rank order,
    rounded once (the oracle's definition, bit-exact)."""
    s = count * 2
    sb, rb = send.view(torch.bfloat16), recv.view(torch.bfloat16)
    for j in range(n):
        sb[j * count:(j + 1) * count].copy_(bf16_chunk(rank, j, count))
    acc = None
    for i in range(n):
        x = bf16_chunk(i, rank, count).float()
        acc = x if acc is None else acc + x
    exp = acc.to(torch.bfloat16)
    out = {"us": {}, "busbw": {}}
    iters = int(max(5, min(100, 4e8 / max(1, (n - 1) * s))))

    def ours():
        cc.reduce_scatter(comms, [send], [recv], count, dtype="bf16", op="sum", impl="sm", streams=stream)

    ok, err = True, None
    try:
        recv.fill_(0)
        torch.cuda.synchronize()
        ours()
        stream.synchronize()
        ok = bool(torch.equal(rb, exp))
        err = None if ok else "parity failed"
    except Exception as e:  # noqa: BLE001
        ok, err = False, str(e)[:160]
    if all_true(ok):
        for _ in range(2):
            ours()
        stream.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            ours()
        e1.record(stream)
        stream.synchronize()
        ms = max_all(e0.elapsed_time(e1) / iters)
        out["us"]["sm"] = round(ms * 1e3, 2)
        out["busbw"]["sm"] = round(busbw(n, s, ms), 2)
    else:
        out["errors"] = {"sm": err or "failed on another rank"}
    if nccl is not None:
        STATE["phase"] = "nccl reduce_scatter"
        with torch.cuda.stream(stream):
            for _ in range(3):
                dist.reduce_scatter_tensor(rb, sb, op=dist.ReduceOp.SUM, group=nccl)
            stream.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(iters):
                dist.reduce_scatter_tensor(rb, sb, op=dist.ReduceOp.SUM, group=nccl)
            e1.record(stream)
        stream.synchronize()
        t = max_all(e0.elapsed_time(e1) / iters)
        out["us"]["nccl"] = round(t * 1e3, 2)
        out["busbw"]["nccl"] = round(busbw(n, s, t), 2)
        if "sm" in out["us"]:
            out["best_over_nccl_time"] = round(out["us"]["sm"] / out["us"]["nccl"], 3)
    return out


# ---------------------------------------------------------------------------
# interference (BASELINE.json configs[4]): FSDP-style all-gather of bf16
# shards beside back-to-back cuBLAS bf16 GEMMs, one rank per GPU
# ---------------------------------------------------------------------------


def run_interference(world, rank, dev, nccl, stream, args, out):
    n = world
    s = int(args.interference_chunk)
    N = 8192
    iters = 40
    comms = cc.Comm.init_ranks(n, rank, 1, dev, cc.torch_exchange())
    win = torch.empty((n + 1) * s, dtype=torch.uint8, device="cuda")
    comms[0].register(win)
    send, recv = win[:s], win[s:(n + 1) * s]
    exp = torch.empty(n * s, dtype=torch.uint8, device="cuda")
    fill_and_expect("allgather", s, n, [rank], [send], [exp], "cuda")
    a = torch.randn(N, N, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, N, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(N, N, device="cuda", dtype=torch.bfloat16)
    gs = torch.cuda.Stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def gemms(k):
        with torch.cuda.stream(gs):
            for _ in range(k):
                torch.matmul(a, b, out=c)

    gemms(5)
    gs.synchronize()
    g0, g1 = ev(), ev()
    g0.record(gs)
    gemms(iters)
    g1.record(gs)
    gs.synchronize()
    gemm_alone = max_all(g0.elapsed_time(g1) / iters)
    out.update({"workload": f"all-gather of {s >> 20} MiB bf16 shards x {n} GPUs beside cuBLAS bf16 {N}^3 "
                            f"GEMMs (one rank per GPU)", "gemm_alone_ms": round(gemm_alone, 4),
                "gemm_alone_tflops": round(2 * N ** 3 / gemm_alone / 1e9, 1), "impls": {}})
    # prelaunch last (cross-device conditional graphs: the least exercised form)
    cands = ["pcpy", "b2b", "hybrid", "sm"] + (["nccl"] if nccl is not None else []) + ["prelaunch_pcpy"]
    for impl in cands:
        STATE["phase"] = f"interference {impl}"
        plan, ok, err = None, True, None
        if impl != "nccl":
            try:
                recv.fill_(0xA5)
                torch.cuda.synchronize()
                plan = cc.Plan(comms, "allgather", [send], [recv], s, impl=impl)
            except cc.CecollError as e:
                ok, err = False, str(e)[:160]
        if not all_true(ok):
            out["impls"][impl] = {"error": err or "failed on another rank"}
            continue

        def coll():
            if plan is None:
                dist.all_gather_into_tensor(recv, send, group=nccl)
            else:
                plan.launch(stream)

        with torch.cuda.stream(stream):
            coll()
        stream.synchronize()
        if plan is not None:
            plan.disarm()
        ok = all_true(bool(torch.equal(recv, exp)))
        if not ok:
            out["impls"][impl] = {"error": "parity failed"}
            if plan is not None:
                plan.destroy()
            continue
        with torch.cuda.stream(stream):
            for _ in range(2):
                coll()
            stream.synchronize()
            dist.barrier()
            c0, c1 = ev(), ev()
            c0.record(stream)
            for _ in range(5):
                coll()
            c1.record(stream)
        stream.synchronize()
        alone = max_all(c0.elapsed_time(c1) / 5)
        k = int(max(4, min(400, round(iters * gemm_alone / alone))))
        dist.barrier()
        g0, g1, c0, c1 = ev(), ev(), ev(), ev()
        g0.record(gs)
        gemms(iters)
        g1.record(gs)
        with torch.cuda.stream(stream):
            c0.record(stream)
            for _ in range(k):
                coll()
            c1.record(stream)
        gs.synchronize()
        stream.synchronize()
        if plan is not None:
            plan.disarm()
            torch.cuda.synchronize()
            plan.destroy()
        gemm_with = max_all(g0.elapsed_time(g1) / iters)
        coll_with = max_all(c0.elapsed_time(c1) / k)
        out["impls"][impl] = {
            "collective_alone_ms": round(alone, 4), "collective_with_gemm_ms": round(coll_with, 4),
            "collective_busbw_alone_gbs": round(busbw(n, s, alone), 1), "collectives": k,
            "gemm_with_collective_ms": round(gemm_with, 4), "gemm_slowdown": round(gemm_with / gemm_alone, 3),
            "collective_slowdown": round(coll_with / alone, 3)}
    torch.cuda.synchronize()
    dist.barrier()
    quiet_destroy(comms[:1])


def run_sync_chain(world, rank, dev, stream, out):
    """Producer -> collective (simulate_sync_chain, sim.cpp:475-499):
    a bf16 4096^3 GEMM, then an all-gather on the same stream, one rank per
    GPU. overhead = T(chain) - T(GEMM) - T(collective), device time, max over
    ranks: stream-ordered plans (the collective enqueued behind the producer,
    no host in between) against the CPU-forwarded chain (the host waits for
    the GEMM, then issues — the paper's baseline)."""
    n = world
    N = 4096
    a = torch.randn(N, N, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, N, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(N, N, device="cuda", dtype=torch.bfloat16)
    comms = cc.Comm.init_ranks(n, rank, 1, dev, cc.torch_exchange())
    smax = 16 << 20
    win = torch.empty((n + 1) * smax, dtype=torch.uint8, device="cuda")
    comms[0].register(win)

    def timed(fn, iters=10):
        ts = []
        for _ in range(iters + 2):
            stream.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            stream.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts = sorted(ts[2:])
        return max_all(ts[len(ts) // 2])

    def gemm():
        with torch.cuda.stream(stream):
            torch.matmul(a, b, out=c)

    t_gemm = timed(gemm)
    out.update({"gemm": f"bf16 {N}^3", "gemm_ms": round(t_gemm, 4), "cases": []})
    for s in (1 << 20, smax):
        send, recv = win[:s], win[s:(n + 1) * s]
        for mode, impl in (("stream", "sm"), ("stream", "pcpy"), ("host", "sm")):
            ok, err, plan = True, None, None
            try:
                plan = cc.Plan(comms, "allgather", [send], [recv], s, impl=impl)
            except cc.CecollError as e:
                ok, err = False, str(e)[:120]
            if not all_true(ok):
                out["cases"].append({"s": s, "mode": mode, "impl": impl, "error": err or "another rank"})
                continue

            def coll():
                plan.launch(stream)

            def chain():
                gemm()
                if mode == "host":
                    stream.synchronize()  # the CPU observes the GEMM, then issues
                coll()

            t_coll = timed(coll)
            t_chain = timed(chain)
            plan.destroy()
            out["cases"].append({"s": s, "mode": mode, "impl": impl, "collective_ms": round(t_coll, 4),
                                 "chain_ms": round(t_chain, 4),
                                 "overhead_us": round((t_chain - t_gemm - t_coll) * 1e3, 2)})
    torch.cuda.synchronize()
    dist.barrier()
    quiet_destroy(comms[:1])


# ---------------------------------------------------------------------------
# experiments: design questions only a multi-GPU node can answer, run after
# every main result is in the line (a hang here prints the line and exits 0)
# ---------------------------------------------------------------------------

EXPERIMENTS = [
    # (name, kind, impl, environment read at plan creation)
    ("sm_peer_tma", "alltoall", "sm", {"CECOLL_PEER_TMA": "1"}),
    ("sm_peer_tma", "allgather", "sm", {"CECOLL_PEER_TMA": "1"}),
    ("pcpy_memop_signals", "alltoall", "pcpy", {"CECOLL_REMOTE_SIGNAL": "memop"}),
    ("b2b_memop_signals", "alltoall", "b2b", {"CECOLL_REMOTE_SIGNAL": "memop"}),
    ("pcpy_memop_signals", "allgather", "pcpy", {"CECOLL_REMOTE_SIGNAL": "memop"}),
]


def guarded_trial(comms, kind, impl, sends, recvs, expects, s, iters, stream):
    """try_impl's protocol with every local failure caught, so every rank runs
    the same sequence of gloo collectives whatever happens on one of them."""
    plan, ok, err, ms = None, True, None, float("inf")
    try:
        for r in recvs:
            r.fill_(0xA5)
        torch.cuda.synchronize()
        plan = cc.Plan(comms, kind, sends, recvs, s, impl=impl)
    except Exception as e:  # noqa: BLE001
        ok, err = False, str(e)[:160]
    ok = all_true(ok)
    if ok:
        try:
            plan.launch(stream)
            stream.synchronize()
            ok = all(bool(torch.equal(r, e)) for r, e in zip(recvs, expects))
            err = None if ok else "parity failed"
        except Exception as e:  # noqa: BLE001
            ok, err = False, str(e)[:160]
    ok = all_true(ok)
    if ok:
        try:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(2):
                plan.launch(stream)
            stream.synchronize()
            e0.record(stream)
            for _ in range(iters):
                plan.launch(stream)
            e1.record(stream)
            stream.synchronize()
            ms = e0.elapsed_time(e1) / iters
        except Exception as e:  # noqa: BLE001
            ok, err = False, str(e)[:160]
    ok = all_true(ok)
    ms = max_all(ms)
    try:
        if plan is not None:
            plan.destroy()
    except Exception:  # noqa: BLE001
        pass
    return ({"ms": round(ms, 4), "busbw_gbs": round(busbw(comms[0].nranks, s, ms), 2)}
            if ok else {"error": err or "failed on another rank"})


def run_experiments(comms, sets, n, s, my_ranks, stream, out):
    sends, recvs = sets[0]
    expects = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in comms]
    filled = None
    for name, kind, impl, env in EXPERIMENTS:
        STATE["phase"] = f"experiments {name} {kind}"
        if filled != kind:
            fill_and_expect(kind, s, n, my_ranks, sends, expects, "cuda")
            torch.cuda.synchronize()
            filled = kind
        snd = [t[:s] for t in sends] if kind == "allgather" else sends
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            res = guarded_trial(comms, kind, impl, snd, recvs, expects, s, 10, stream)
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        out[f"{name}/{kind}"] = res


def run_ce_share_experiment(world, rank, dev, out):
    """Copy-engine sharing over NVLink (the reference models
    max-min fair flows, sim.cpp:124-179): rank 0 releases k peer copies of
    64 MiB at once (one stream each) from its GPU to k peers, and k copies to
    one peer, and records each copy's completion. On the one-GPU boxes the
    host link serialises same-direction copies (profiles/ce_share_r02.json);
    this measures the same on NVLink. The other ranks wait at the barrier."""
    res = {}
    out["ce_share_nvlink"] = res
    try:
        ng = torch.cuda.device_count()
        if rank == 0 and ng >= 2:
            n = 64 << 20
            src = torch.empty(n, dtype=torch.uint8, device=f"cuda:{dev}")
            cases = {f"{k}_peers": [(dev + 1 + i) % ng for i in range(k)] for k in (1, 2, 4, ng - 1) if k <= ng - 1}
            cases["4_to_one_peer"] = [(dev + 1) % ng] * 4
            for name, peers in cases.items():
                dsts = [torch.empty(n, dtype=torch.uint8, device=f"cuda:{p}") for p in peers]
                streams = [torch.cuda.Stream(device=dev) for _ in peers]
                best = None
                for _ in range(3):
                    torch.cuda.synchronize(dev)
                    go = torch.cuda.Event(enable_timing=True)
                    ends = [torch.cuda.Event(enable_timing=True) for _ in peers]
                    gate = torch.cuda.Stream(device=dev)
                    with torch.cuda.stream(gate):
                        torch.cuda._sleep(2_000_000)
                        go.record(gate)
                    for d, s, e in zip(dsts, streams, ends):
                        s.wait_event(go)
                        with torch.cuda.stream(s):
                            d.copy_(src, non_blocking=True)
                            e.record(s)
                    for s in streams:
                        s.synchronize()
                    t = [go.elapsed_time(e) for e in ends]
                    if best is None or max(t) < max(best):
                        best = t
                res[name] = {"peers": peers, "done_ms": [round(x, 3) for x in best],
                             "aggregate_gbs": round(len(peers) * n / max(best) / 1e6, 1),
                             "single_copy_gbs": round(n / min(best) / 1e6, 1)}
                del dsts
    except Exception as e:  # noqa: BLE001
        res["error"] = str(e)[:200]
    finally:
        torch.cuda.synchronize()
        dist.barrier()


def run_tune_experiment(world, rank, dev, stream, out):
    """cecoll_tune on the node (csrc/tune.cpp): one rank per GPU, every
    applicable implementation at 4 KiB-16 MiB chunks, device time max over
    ranks and processes; the measured winner grid that replaces the static
    multi-device guess in program.cpp select. Reports the
    installed table, every candidate's time, and whether every process
    installed the same table."""
    res = {}
    out["tune"] = res
    comms = cc.Comm.init_ranks(world, rank, 1, dev, cc.torch_exchange())
    try:
        t0 = time.time()
        cc.tune(comms, max_chunk=16 << 20, streams=stream)
        table = comms[0].tuned_table()
        tables = [None] * world
        dist.all_gather_object(tables, table)
        res["seconds"] = round(time.time() - t0, 1)
        res["table"] = [f"{k} {s} {i}" for k, s, i in table]
        res["same_on_every_rank"] = all(t == table for t in tables)
        res["us"] = {f"{k} {s}": v["us"] for (k, s), v in comms[0].tune_report().items()}
        res["static"] = {f"{k} {s}": cc.select(k, s, world, world) for k, s, _ in table}
    except Exception as e:  # noqa: BLE001
        res["error"] = str(e)[:200]
    finally:
        torch.cuda.synchronize()
        dist.barrier()
        quiet_destroy(comms)


def run_mc_experiment(world, rank, dev, stream, out):
    """NVLS multicast all-gather (include/cecoll.h cecoll_mc_*):
    one rank per GPU, window creation and every collective under consensus,
    parity against the seeded expectation, then timing. Last experiment: the
    least tested path in the library (never executed on a box that accepts
    multicast objects)."""
    n = world
    cap = 64 << 20
    res = {}
    out["nvls_allgather"] = res
    comms = cc.Comm.init_ranks(n, rank, 1, dev, cc.torch_exchange())
    win, ok, err = None, True, None
    try:
        win = cc.McWindow(comms[0], cap)
        res["handle_type"] = win.handle_type
    except Exception as e:  # noqa: BLE001
        ok, err = False, str(e)[:200]
    if not all_true(ok):
        res["error"] = err or "window creation failed on another rank"
        quiet_destroy(comms[:1])
        return
    send = torch.empty(cap, dtype=torch.uint8, device="cuda")
    exp = torch.empty(n * cap, dtype=torch.uint8, device="cuda")
    for s in (1 << 20, 16 << 20, 64 << 20):
        fill_and_expect("allgather", s, n, [rank], [send], [exp], "cuda")
        torch.cuda.synchronize()
        ok, err = True, None
        try:
            win.allgather(send, s, stream)
            stream.synchronize()
            ok = bool(torch.equal(win.recv[:n * s], exp[:n * s]))
            err = None if ok else "parity failed"
        except Exception as e:  # noqa: BLE001
            ok, err = False, str(e)[:160]
        if not all_true(ok):
            res[str(s)] = {"error": err or "failed on another rank"}
            break
        iters = int(max(5, min(100, 4e8 / max(1, (n - 1) * s))))
        for _ in range(2):
            win.allgather(send, s, stream)
        stream.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            win.allgather(send, s, stream)
        e1.record(stream)
        stream.synchronize()
        ms = max_all(e0.elapsed_time(e1) / iters)
        res[str(s)] = {"us": round(ms * 1e3, 2), "busbw_gbs": round(busbw(n, s, ms), 2)}
    torch.cuda.synchronize()
    dist.barrier()
    try:
        win.destroy()
    except Exception:  # noqa: BLE001
        pass
    quiet_destroy(comms[:1])
