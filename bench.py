"""cecoll benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1]): all-to-all over 8 ranks with a 64 MiB
send buffer per rank (per-peer chunk s = 8 MiB, SURVEY.md §8 sizing). With
one GPU the 8 ranks are co-resident on it (comm_init_all with a repeated
device), so every chunk transfer is an HBM->HBM copy through the executor.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--algo auto|sm|pcpy|b2b|prelaunch_pcpy|...] [--sweep]

A step is one collective over the synthetic inputs. `value` is the
nccl-tests bus bandwidth of the 8-rank collective, busBW = (n-1)*s/t, with
inputs resident in HBM; `e2e` is the same metric through the public API with
the inputs copied from pinned host memory and the results copied back inside
the timed region. `--impl reference` times the reference's CPU path (the
reference's own compile() from oracle/_ref plus the byte executor) on the
host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import paper_2511_06605_b200 as cc  # noqa: E402  (sets CUDA_DEVICE_MAX_CONNECTIONS first)

NRANKS = 8
SEND_PER_RANK = 64 << 20
CHUNK = SEND_PER_RANK // NRANKS  # s = 8 MiB
METRIC = "alltoall_busbw_8ranks_x_64MiB"
WORKLOAD = "alltoall, 8 ranks x 64 MiB send/rank (s = 8 MiB per peer), BASELINE configs[1]"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def load_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_items_kernel.json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:  # noqa: BLE001
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index=0):
        self.proc = None
        self.lines = []
        self.gpu = gpu_index

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        """Median SM clock over samples taken under load (power above idle +
        100 W; all samples if none qualify) and every throttle reason seen."""
        rows, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[3])))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": 0}
        idle = min(p for _, p in rows)
        loaded = [c for c, p in rows if p > idle + 100] or [c for c, _ in rows]
        loaded.sort()
        return {"sm_mhz": loaded[len(loaded) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(rows), "samples_under_load": len(loaded),
                "power_w_max": max(p for _, p in rows)}


def busbw(n, s, seconds):
    return (n - 1) * s / seconds / 1e9


def bench_config():
    """The workload, identical in both arms' lines (the driver compares the
    `config` dicts); everything arm-specific goes under `details`."""
    return {"workload": WORKLOAD, "ranks": NRANKS, "chunk_bytes": CHUNK}


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU path on the host cores
# ---------------------------------------------------------------------------


def cpu_reference_step(kind="alltoall", n=NRANKS, s=CHUNK, impl="pcpy", threads=None):
    """One CPU collective over the full workload with every host thread;
    returns (seconds, kind, threads, sample)."""
    import ctypes as C

    import numpy as np

    from oracle import oracle as ora

    threads = threads or os.cpu_count() or 1
    in_bytes = s if kind == "allgather" else n * s
    ins = [ora.splitmix_pattern(in_bytes, r) for r in range(n)]
    outs = [np.empty(n * s, dtype=np.uint8) for _ in range(n)]
    if os.path.exists(ora.REF_LIB):
        R = ora.Reference()
        R.L.ref_execute_mt.argtypes = [C.c_char_p, C.c_char_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
        ptr_in = ora._ptrs(ins)
        ptr_out = ora._ptrs(outs)

        def once():
            rc = R.L.ref_execute_mt(kind.encode(), impl.encode(), s, n, ptr_in, ptr_out, threads)
            assert rc == 0

        label = "reference"
        what = "the reference's compile() (oracle/_ref) + byte executor, queues over host threads"
    else:
        O = ora.Oracle()

        def once():
            O.reference_result(kind, s, n, ins, outs, threads)

        label = "port"
        what = "oracle restatement (oracle/cecoll_oracle.c), destinations over host threads"
    once()  # warm the pages
    best = float("inf")
    for _ in range(3):
        t0 = time.perf_counter()
        once()
        best = min(best, time.perf_counter() - t0)
    return best, label, threads, f"{kind} {impl} n={n} s={s}: full workload, {what}, best of 3"


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    times = []
    for _ in range(args.warmup):
        cpu_reference_step()
    label, cores, sample = None, 1, ""
    for _ in range(args.steps):
        dt, label, cores, sample = cpu_reference_step()
        times.append(dt)
    t = sum(times) / len(times)
    v = busbw(NRANKS, CHUNK, t)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(v, 3),
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic splitmix64 pattern",
        "config": bench_config(),
        "details": {"device": "host CPU"},
        "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": cores, "kind": label, "sample": sample},
        "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def run_ours(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import bench_mgpu

        return bench_mgpu.run(args, sys.modules[__name__])
    dev = 0
    torch.cuda.set_device(dev)
    n, s = NRANKS, CHUNK
    comms = cc.Comm.init_all([dev] * n)
    stream = torch.cuda.Stream()
    g = torch.Generator(device="cuda").manual_seed(0)
    sends = [torch.randint(0, 256, (n * s,), dtype=torch.uint8, device="cuda", generator=g) for _ in range(n)]
    recvs = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
    impl = args.algo
    chosen = cc.select("alltoall", s, n, 1) if impl == "auto" else impl
    torch.cuda.synchronize()

    def step():
        cc.all_to_all(comms, sends, recvs, s, impl=chosen, streams=stream)

    with torch.cuda.stream(stream):
        for _ in range(max(3, args.warmup)):
            step()
    torch.cuda.synchronize()
    c0 = comms[0].counters()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    # nvidia-smi samples every 100 ms while the timed region (a few ms) runs
    # and then while the same step keeps running for the >= 1.5 s NVML energy
    # loop, so the clocks reported are clocks under this load.
    with ClockSampler(dev) as clocks:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        c1 = comms[0].counters()
        energy = None if args.no_energy else measure_energy(step, stream, n, s)
    ms = e0.elapsed_time(e1) / args.steps
    value = busbw(n, s, ms / 1e3)
    plan_info = comms[0].last_plan_info()  # the plan the timed steps ran

    # Parity of the timed buffers against the definition: every chunk of every
    # rank, compared on the device (recv_j[i] = send_i[j], compiler.cpp:156-157).
    ok = all(torch.equal(recvs[j][i * s:(i + 1) * s], sends[i][j * s:(j + 1) * s])
             for i in range(n) for j in range(n))

    # Roofline of the dominant kernel: one launch moves every chunk (n*n*s
    # bytes read + written; the local placement included).
    peak, peak_kind = load_peaks()
    alg_bytes = 2 * n * n * s
    achieved = alg_bytes / (ms / 1e3) / 1e9
    kernels_per_step = (c1["kernels"] - c0["kernels"]) / args.steps
    graphs_per_step = (c1["graph_launches"] - c0["graph_launches"]) / args.steps

    # e2e: pinned host inputs -> HBM -> collective -> HBM -> pinned host results.
    # Every rank's buffer is a row of one [n, n*s] tensor (host and device), so
    # each direction of a step is ONE 512 MiB copy: one large DMA per direction
    # runs the PCIe link closer to its duplex peak than eight 64 MiB copies
    # (10.93 vs 11.36 ms, gpurun_out/pcie5 / pcie_probe4, profiles/pcie_r02.txt).
    host_in_all = torch.empty((n, n * s), dtype=torch.uint8, pin_memory=True)
    host_in = list(host_in_all.unbind(0))
    for h, d in zip(host_in, sends):
        h.copy_(d)
    # Pipeline fill (the first step's inputs) and drain (the last step's
    # results) are paid once per timed window: more steps amortise them.
    e2e_steps = max(args.e2e_steps, args.steps)
    # Two device buffer sets so that step k's device->host copy overlaps step
    # k+1's host->device copy (PCIe is full duplex); every step still copies
    # its inputs in and its results out inside the timed region.
    dev_sets = [(torch.empty((n, n * s), dtype=torch.uint8, device="cuda"),
                 torch.empty((n, n * s), dtype=torch.uint8, device="cuda")) for _ in range(2)]
    sets = [(list(a.unbind(0)), list(b.unbind(0))) for a, b in dev_sets]
    host_out_all = [torch.empty((n, n * s), dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    host_outs = [list(h.unbind(0)) for h in host_out_all]
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    in_ready = [torch.cuda.Event() for _ in range(2)]
    coll_done = [torch.cuda.Event() for _ in range(2)]
    out_done = [torch.cuda.Event() for _ in range(2)]
    for ev in coll_done + out_done:
        ev.record(stream)

    def e2e_step(k):
        b = k % 2
        sd, rv = sets[b]
        h2d_s.wait_event(coll_done[b])  # collective k-2 has read sd
        with torch.cuda.stream(h2d_s):
            dev_sets[b][0].copy_(host_in_all, non_blocking=True)
        in_ready[b].record(h2d_s)
        stream.wait_event(in_ready[b])
        stream.wait_event(out_done[b])  # results k-2 have left rv
        cc.all_to_all(comms, sd, rv, s, impl=chosen, streams=stream)
        coll_done[b].record(stream)
        d2h_s.wait_event(coll_done[b])
        with torch.cuda.stream(d2h_s):
            host_out_all[b].copy_(dev_sets[b][1], non_blocking=True)
        out_done[b].record(d2h_s)

    for k in range(2):
        e2e_step(k)
    torch.cuda.synchronize()
    # Cold window: the pipeline starts empty (the first step's inputs cross
    # PCIe alone) and is drained at the end (the last results alone).
    e0.record(h2d_s)
    k = 2
    for _ in range(e2e_steps):
        e2e_step(k)
        k += 1
    e1.record(d2h_s)
    torch.cuda.synchronize()
    cold_ms = e0.elapsed_time(e1) / e2e_steps
    # Steady window: the same loop with the pipeline kept full across the
    # window's edges — the step rate of a long-running job. Every step still
    # copies its inputs in and its results out; the window spans K result
    # copies and the K input copies they depend on.
    for _ in range(2):
        e2e_step(k)
        k += 1
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(d2h_s)
    for _ in range(e2e_steps):
        e2e_step(k)
        k += 1
    s1.record(d2h_s)
    torch.cuda.synchronize()
    e2e_ms = s0.elapsed_time(s1) / e2e_steps
    e2e_value = busbw(n, s, e2e_ms / 1e3)
    e2e_ok = all(torch.equal(host_outs[(k - 1) % 2][j][i * s:(i + 1) * s], host_in[i][j * s:(j + 1) * s])
                 for i in range(n) for j in range(n))
    floor_ms = pcie_floor_ms([host_in_all], [host_out_all[0]], [dev_sets[0][0]], [dev_sets[0][1]], h2d_s, d2h_s)

    cpu = None
    if not args.no_cpu_baseline:
        dt, label, cores, sample = cpu_reference_step()
        cpu = {"value": round(busbw(n, s, dt), 3), "unit": "GB/s", "cores": cores, "kind": label,
               "sample": sample + f"; {dt * 1e3:.1f} ms"}

    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GB/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic (torch.randint bytes)",
        "config": bench_config(),
        "details": {
            "ranks_per_gpu": n,
            "impl": chosen,
            "l2": "inputs larger than L2 (1 GiB touched per step vs 126 MB L2)",
            "aggregate_gbs": round(n * value, 3),
            "algbw_gbs": round(n * s / (ms / 1e3) / 1e9, 3),
            "plan": plan_info,
        },
        "parity_ok": bool(ok),
        "roofline": {
            "bound": "hbm",
            "achieved": round(achieved, 1),
            "peak": peak,
            "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            "traffic": load_traffic(),
            "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu "
                              "--set full capture of this kernel (profiles/ncu_items_kernel.json), not measured "
                              "in this run",
            "peak_source": peak_kind + " hbm_gbs (copy, read+write)",
            "algorithmic_bytes_per_launch": alg_bytes,
            "busbw_bound_gbs": round(busbw(n, s, alg_bytes / (peak * 1e9)), 1),
        },
        "cpu_baseline": cpu,
        "e2e": {"value": round(e2e_value, 3), "unit": "GB/s", "h2d_bytes_per_step": n * n * s,
                "d2h_bytes_per_step": n * n * s, "ms_per_step": round(e2e_ms, 3), "parity_ok": bool(e2e_ok),
                "steps": e2e_steps, "window": "steady state (pipeline full at both edges)",
                "cold_ms_per_step": round(cold_ms, 3),
                "cold_value": round(busbw(n, s, cold_ms / 1e3), 3),
                "floor_ms": round(floor_ms, 3), "vs_floor": round(e2e_ms / floor_ms, 4),
                "floor_value": round(busbw(n, s, floor_ms / 1e3), 3),
                "pipeline": "double-buffered: H2D of step k+1 overlaps D2H of step k; one 512 MiB copy per "
                            "direction per step (the ranks' buffers are rows of one [n, n*s] tensor)",
                "bound_note": "host-bound: 512 MiB host->device and 512 MiB device->host per step over one "
                              "x16 link, i.e. 1 GiB of host memory traffic per step, the same the CPU arm "
                              "moves (profiles/host_mem_probe_r02.txt). floor_ms is measured in this run: the same bytes copied both ways "
                              "at once on the same streams with no collective, 6 steps back to back, per "
                              "step (best of 3 loops)"},
        "gpu_launches": int(round((kernels_per_step + 4 * graphs_per_step) * args.steps)),
        "energy": energy,
        "clocks": clocks.summary(),
    }
    err = comms[0].async_error()  # a device-side poll timeout anywhere in the run (none expected)
    if err is not None:
        line["async_error"] = str(err)[:200]
    print(json.dumps(line), flush=True)
    try:
        cc.destroy_all(comms)
    except cc.CecollError:
        pass  # already reported in the line


def pcie_floor_ms(host_in, host_out, dev_in, dev_out, h2d_s, d2h_s, reps=3, steps=6):
    """Per-step floor of the e2e leg: the step's host->device and
    device->host bytes moved at the same time (full duplex) on the e2e's own
    streams and buffers, with no collective, `steps` steps back to back so
    the link is as continuously busy as in the e2e's steady state; the best
    of `reps` such loops, per step (CUDA events)."""
    import torch

    best = float("inf")
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        e0.record(cur)
        h2d_s.wait_event(e0)
        d2h_s.wait_event(e0)
        for _ in range(steps):
            with torch.cuda.stream(h2d_s):
                for h, d in zip(host_in, dev_in):
                    d.copy_(h, non_blocking=True)
            with torch.cuda.stream(d2h_s):
                for h, d in zip(host_out, dev_out):
                    h.copy_(d, non_blocking=True)
        cur.wait_stream(h2d_s)
        cur.wait_stream(d2h_s)
        e1.record(cur)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / steps)
    return best


def measure_energy(step, stream, n, s, seconds=1.5, dev=0):
    """NVML energy per transferred GB over a >= `seconds` loop of `step`
    (J/GB = dE / (n(n-1)s bytes per collective x collectives / 1e9))."""
    try:
        import pynvml
    except Exception:  # noqa: BLE001
        return None
    import torch

    try:
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        count = 0
        while time.perf_counter() - t0 < seconds:
            for _ in range(20):
                step()
            count += 20
            stream.synchronize()
        torch.cuda.synchronize()
        e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        dt = time.perf_counter() - t0
        joules = (e1 - e0) / 1e3
        gb = n * (n - 1) * s * count / 1e9
        return {"j_per_gb": round(joules / gb, 5), "joules": round(joules, 3), "seconds": round(dt, 3),
                "avg_power_w": round(joules / dt, 1), "collectives": count,
                "note": "NVML total energy of the GPU over the loop / link-equivalent bytes n(n-1)s"}
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)}


def run_interference(args):
    """C4 (BASELINE configs[4]): an all-gather loop of bf16 shards beside a
    back-to-back cuBLAS bf16 8192^3 GEMM; reports the GEMM slowdown and the
    collective slowdown per implementation (ranks co-resident on one GPU)."""
    import torch

    torch.cuda.set_device(0)
    n = args.ranks
    s = args.interference_chunk
    comms = cc.Comm.init_all([0] * n)
    elems = s // 2
    g = torch.Generator(device="cuda").manual_seed(0)
    sends = [torch.randn(elems, generator=g, device="cuda").to(torch.bfloat16) for _ in range(n)]
    recvs = [torch.empty(n * elems, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    N = 8192
    a = torch.randn(N, N, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, N, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(N, N, device="cuda", dtype=torch.bfloat16)
    # --gemm-priority high: the GEMM stream gets the highest stream priority,
    # the collective the lowest (the block scheduler then prefers GEMM CTAs).
    gemm_s = torch.cuda.Stream(priority=-5 if args.gemm_priority == "high" else 0)
    coll_s = torch.cuda.Stream()
    flops = 2 * N ** 3

    def gemm_loop(iters):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
        with torch.cuda.stream(gemm_s):
            for e0, e1 in ev:
                e0.record(gemm_s)
                torch.matmul(a, b, out=c)
                e1.record(gemm_s)
        return ev

    def times(ev):
        return sorted(e0.elapsed_time(e1) for e0, e1 in ev)

    # GEMM alone
    gemm_loop(5)
    torch.cuda.synchronize()
    ev_alone = gemm_loop(args.gemm_iters)
    torch.cuda.synchronize()
    alone = times(ev_alone)
    gemm_alone_ms = alone[len(alone) // 2]
    out = {"workload": f"all-gather {n} ranks x {s >> 20} MiB bf16 shards (co-resident on 1 GPU) beside "
                       f"cuBLAS bf16 {N}^3 GEMM", "gemm_alone_ms": round(gemm_alone_ms, 4),
           "gemm_alone_tflops": round(flops / gemm_alone_ms / 1e9, 1), "impls": {}}
    host_recvs = None
    for spec in args.interference_impls.split(","):
        # "impl[@budget][:host]": budget = the world's SM budget (max CTAs per
        # kernel, cecoll_comm_set_sm_budget) for this plan; ":host" = recv
        # buffers in pinned host memory, so the copy-engine lanes run on the
        # copy engines (device-local copies run on SMs).
        impl, _, where = spec.partition(":")
        impl, _, budget = impl.partition("@")
        budget = int(budget or 0)
        rb, sb, cs, ce = recvs, sends, s, elems
        if where == "host":  # PCIe-bound: a smaller shard keeps the pinned footprint at n*n*chunk
            cs = args.interference_host_chunk
            ce = cs // 2
            if host_recvs is None:
                host_recvs = [torch.empty(n * ce, dtype=torch.bfloat16, pin_memory=True) for _ in range(n)]
            rb, sb = host_recvs, [t[:ce] for t in sends]
        comms[0].set_sm_budget(budget)
        plan = cc.Plan(comms, "allgather", sb, rb, cs, impl=impl)
        comms[0].set_sm_budget(0)
        impl = spec
        # collective alone
        for _ in range(3):
            plan.launch(coll_s)
        coll_s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(coll_s)
        for _ in range(5):
            plan.launch(coll_s)
        e1.record(coll_s)
        coll_s.synchronize()
        coll_alone = e0.elapsed_time(e1) / 5
        # Concurrent window: the GEMM stream holds args.gemm_iters GEMMs; the
        # collective stream is kept busy (<= 3 in flight) until the last GEMM
        # ends, so every GEMM overlaps collectives. Rates are taken inside the
        # window: GEMM time = GEMM window / iters; collective time = the
        # collectives that finished inside the window.
        g_start, g_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        coll_ev = []
        g_start.record(gemm_s)
        with torch.cuda.stream(gemm_s):
            for _ in range(args.gemm_iters):
                torch.matmul(a, b, out=c)
        g_end.record(gemm_s)
        while True:
            if len(coll_ev) >= 3:
                coll_ev[-3][1].synchronize()
            e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e_a.record(coll_s)
            plan.launch(coll_s)
            e_b.record(coll_s)
            coll_ev.append((e_a, e_b))
            if g_end.query():
                break
        coll_s.synchronize()
        gemm_s.synchronize()
        info = plan.info()
        plan_info_summary = {"movers": [u["mover"] for u in info["units"]], "grid": [u["grid"] for u in info["units"]],
                             "ce_lanes": [u["ce_lanes"] for u in info["units"]], "recorded": info["recorded"],
                             "graph_fallback": info["graph_fallback"]}
        plan.destroy()
        torch.cuda.synchronize()
        window = g_start.elapsed_time(g_end)
        gemm_with = window / args.gemm_iters
        inside = [(a_, b_) for a_, b_ in coll_ev if g_start.elapsed_time(b_) <= window and
                  g_start.elapsed_time(a_) >= 0]
        if len(inside) >= 2:
            coll_with = inside[0][0].elapsed_time(inside[-1][1]) / len(inside)
        else:
            coll_with = None
        if where == "host":  # parity of the host-resident result (every rank's recv = all shards)
            want = torch.cat([t.cpu() for t in sb])
            parity = all(torch.equal(h, want) for h in rb)
        else:
            parity = all(torch.equal(rb[j][i * ce:(i + 1) * ce], sb[i]) for i in range(n) for j in range(n))
        out["impls"][impl] = {
            "parity_ok": bool(parity),
            "sm_budget": budget,
            "recv": "pinned host" if where == "host" else "device",
            "chunk_bytes": cs,
            "plan": plan_info_summary,
            "collective_alone_ms": round(coll_alone, 4),
            "collective_with_gemm_ms": None if coll_with is None else round(coll_with, 4),
            "collective_slowdown": None if coll_with is None else round(coll_with / coll_alone, 3),
            "collectives_in_window": len(inside),
            "gemm_with_collective_ms": round(gemm_with, 4),
            "gemm_slowdown": round(gemm_with / gemm_alone_ms, 3),
            "gemm_tflops_with_collective": round(flops / gemm_with / 1e9, 1),
        }
        print(impl, out["impls"][impl], flush=True)
    print(json.dumps(out), flush=True)
    if args.interference_out:
        with open(args.interference_out, "w") as f:
            json.dump(out, f, indent=1)
    cc.destroy_all(comms)


def run_sweep_rs(args):
    """Reduce-scatter sweep (bf16 sum, co-resident ranks): busBW = (n-1)*chunk/t
    (nccl-tests convention) and HBM roofline of the SM path (n+1 chunk
    transfers per rank: n reads and one write)."""
    import torch

    n = args.ranks
    torch.cuda.set_device(0)
    comms = cc.Comm.init_all([0] * n)
    peak, _ = load_peaks()
    stream = torch.cuda.Stream()
    rows = []
    for count in [2048 << (2 * k) for k in range(9)]:  # 4 KiB .. 256 MiB bf16 chunks
        s = count * 2
        sends = [torch.randn(n * count, device="cuda").to(torch.bfloat16) for _ in range(n)]
        recvs = [torch.empty(count, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
        torch.cuda.synchronize()  # inputs written on torch's stream, collectives on `stream`
        for impl in [i for i in ("sm", "pcpy", "b2b", "prelaunch_pcpy")
                     if not args.sweep_impls or i in args.sweep_impls.split(",")]:
            def call():
                cc.reduce_scatter(comms, sends, recvs, count, dtype="bf16", op="sum", impl=impl, streams=stream)

            for _ in range(3):
                call()
            stream.synchronize()
            iters = int(max(5, min(300, 2e9 / (n * (n + 1) * s))))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(iters):
                call()
            e1.record(stream)
            stream.synchronize()
            ms = e0.elapsed_time(e1) / iters
            hbm = n * (n + 1) * s / (ms / 1e3) / 1e9
            # the bytes this form must move: the SM path reads every rank's
            # chunk in place (n(n+1)s); the copy-engine forms first gather
            # the n(n-1) remote chunks into staging (read + write) and the
            # reduction reads n chunks per rank and writes one ((3n^2 - n)s)
            own = n * (n + 1) * s if impl == "sm" else (3 * n * n - n) * s
            row = {"impl": impl, "collective": "reduce_scatter_bf16_sum", "ranks": n, "size_bytes": s,
                   "total_ns": round(ms * 1e6), "busbw_gbs": round(busbw(n, s, ms / 1e3), 3),
                   "hbm_gbs": round(hbm, 1), "roofline_frac": round(hbm / peak, 4),
                   "own_bytes": own, "roofline_frac_own": round(own / (ms / 1e3) / 1e9 / peak, 4)}
            rows.append(row)
            print(row, flush=True)
        del sends, recvs
        torch.cuda.empty_cache()
    with open(args.sweep_out, "w") as f:
        cols = list(rows[0].keys())
        f.write(",".join(cols) + "\n")
        for r in rows:
            f.write(",".join(str(r[c]) for c in cols) + "\n")
    cc.destroy_all(comms)


def run_sync_chain(args):
    """Producer GEMM -> all-gather synchronisation (simulate_sync_chain,
    sim.cpp:475-499; §4.3). overhead = T(GEMM then collective on one
    stream) - T(GEMM) - T(collective). Modes: `stream` (collective enqueued
    behind the GEMM, no host involvement), `prelaunch` (armed plan triggered
    by a stream write when the GEMM ends), `host` (the host waits for the GEMM
    and then issues the collective: the CPU-forwarded chain of the paper)."""
    import torch

    torch.cuda.set_device(0)
    n = args.ranks
    comms = cc.Comm.init_all([0] * n)
    N = args.sync_gemm
    a = torch.randn(N, N, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, N, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(N, N, device="cuda", dtype=torch.bfloat16)
    S = torch.cuda.Stream()
    res = {"gemm": f"bf16 {N}^3", "ranks": n, "cases": []}

    def timed(fn, iters=20):
        for _ in range(3):
            fn()
        S.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(iters):
            S.synchronize()
            e0.record(S)
            fn()
            e1.record(S)
            S.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        return ts[len(ts) // 2]

    def gemm():
        with torch.cuda.stream(S):
            torch.matmul(a, b, out=c)

    t_gemm = timed(gemm)
    for s in (1 << 20, 16 << 20, 256 << 20):
        sends = [torch.empty(s, dtype=torch.uint8, device="cuda") for _ in range(n)]
        recvs = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
        for mode, impl in (("stream", "sm"), ("stream", "b2b"), ("prelaunch", "prelaunch_b2b"),
                           ("prelaunch", "prelaunch_pcpy"), ("host", "sm")):
            plan = cc.Plan(comms, "allgather", sends, recvs, s, impl=impl)

            def coll():
                plan.launch(S)

            def chain():
                gemm()
                if mode == "host":
                    S.synchronize()  # the CPU observes the GEMM, then issues
                coll()

            t_coll = timed(coll)
            t_chain = timed(chain)
            plan.destroy()
            torch.cuda.synchronize()
            row = {"s": s, "mode": mode, "impl": impl, "gemm_ms": round(t_gemm, 4), "collective_ms": round(t_coll, 4),
                   "chain_ms": round(t_chain, 4), "overhead_us": round((t_chain - t_gemm - t_coll) * 1e3, 2)}
            res["cases"].append(row)
            print(row, flush=True)
        del sends, recvs
        torch.cuda.empty_cache()
    print(json.dumps(res), flush=True)
    with open(args.sync_out, "w") as f:
        json.dump(res, f, indent=1)
    cc.destroy_all(comms)


# ---------------------------------------------------------------------------
# sweep (run_sweep analog, sweep.cpp:71-184): every implementation x size
# ---------------------------------------------------------------------------

def alg_hbm_bytes(kind, impl, s, n):
    """Algorithmic HBM bytes (read + write) of one collective with co-resident
    ranks: the program's account_traffic (verifier.cpp:281-327) plus the local
    placement (verifier.cpp:40-44) for out-of-place programs. The SM path's
    all-gather reads each source once (fan item)."""
    if impl == "sm":
        return (n * s + n * n * s) if kind == "allgather" else 2 * n * n * s
    if impl == "pull":  # n(n-1) chunk copies + the local placement
        return 2 * n * n * s
    if impl == "hybrid":  # CE share: n(n-1) copies; SM share as the SM path; placement
        sm_b = (s * 50 // 100) & ~15
        ce = s - sm_b
        sm_part = (n * sm_b + n * (n - 1) * sm_b) if kind == "allgather" else 2 * n * (n - 1) * sm_b
        return 2 * n * (n - 1) * ce + sm_part + 2 * n * s
    t = cc.Program(kind, impl, s, n).traffic()
    extra = 0 if impl.endswith("swap") else 2 * n * s
    return t["read"] + t["write"] + extra


SWEEP_COLUMNS = ["impl", "api", "collective", "gpus", "size_bytes", "total_ns", "control_ns", "schedule_ns", "copy_ns",
                 "sync_ns", "trigger_ns", "ranks", "isolated_ns", "busbw_gbs", "hbm_gbs", "roofline_frac",
                 "api_calls", "kernels", "graphs", "parity", "host_ns", "traced_ns"]

# Trace-event name prefix -> phase of the reference's model (sim.cpp Phase:
# Control, Schedule, Copy, Sync, Trigger, Poll; Poll is folded into Sync as
# in the CSV schema, sim.cpp:546-569).
_DEVICE_PHASE = {"copy": "copy", "kernel": "copy", "sync": "sync", "poll": "sync", "trigger": "trigger"}
_PHASE_RANK = ["copy", "trigger", "sync"]  # when device spans overlap, the data movement is on the path


def trace_phases(events):
    """Critical-path attribution of one traced collective (phase_breakdown,
    sim.cpp:501-508, on a measured timeline). Every instant between the first
    host submission and the last device command is given one phase: a device
    command in flight (copy > trigger > sync when they overlap); else the
    host submitting (control, or trigger for a prelaunch trigger); else
    nothing in flight — the device waits for submitted work to start
    (schedule: launch latency, doorbells). Returns ({phase: ns}, traced ns)."""
    open_, spans = {}, []
    for e in events:
        key = (e["name"], e["pid"], e["tid"])
        if e["ph"] == "B":
            open_.setdefault(key, []).append(e["ts"])
        elif open_.get(key):
            spans.append((e["name"], e["pid"], open_[key].pop(), e["ts"]))
    dev = [(n.split(":")[0], b, e) for n, pid, b, e in spans if pid >= 0]
    host = [(("trigger" if n.startswith("trigger") else "control"), b, e) for n, pid, b, e in spans if pid < 0]
    if not dev:
        return None, 0.0
    t0 = min([b for _, b, _ in dev] + [b for _, b, _ in host])
    t1 = max(e for _, _, e in dev)
    cuts = sorted({t for _, b, e in dev + host for t in (b, e) if t0 <= t <= t1} | {t0, t1})
    out = {"control": 0.0, "schedule": 0.0, "copy": 0.0, "sync": 0.0, "trigger": 0.0}
    for a, b in zip(cuts, cuts[1:]):
        mid = (a + b) / 2
        act = {_DEVICE_PHASE.get(k, "copy") for k, x, y in dev if x <= mid < y}
        if act:
            ph = next(p for p in _PHASE_RANK if p in act)
        else:
            hs = [k for k, x, y in host if x <= mid < y]
            ph = ("trigger" if "trigger" in hs else "control") if hs else "schedule"
        out[ph] += (b - a) * 1e3  # µs -> ns
    return out, (t1 - t0) * 1e3


def run_sweep(args):
    """CSV with the reference's schema (sim.cpp:546-569) plus measured columns.

    total_ns    device time per collective, back to back (throughput view)
    isolated_ns device time of one collective issued on an idle stream
    control_ns  host time spent inside the API call (the paper's control phase)
    """
    import torch

    from oracle import oracle as ora

    n = args.ranks
    torch.cuda.set_device(0)
    comms = cc.Comm.init_all([0] * n)
    peak, _ = load_peaks()
    stream = torch.cuda.Stream()
    rows = []
    sizes = [4096 << (2 * k) for k in range(10)]  # 4 KiB .. 1 GiB
    if args.sweep_sizes:
        sizes = [int(float(x)) for x in args.sweep_sizes.split(",")]
    out_path = args.sweep_out
    O = ora.Oracle()
    kinds = args.sweep_kinds.split(",") if args.sweep_kinds else ["allgather", "alltoall"]
    for kind in kinds:
        impls = ["sm", "hybrid", "pull"] + cc.IMPLS_FOR[kind]
        if args.sweep_impls:
            impls = [i for i in impls if i in args.sweep_impls.split(",")]
        for s in sizes:
            in_bytes = s if kind == "allgather" else n * s
            if n * (in_bytes + n * s) > args.max_bytes:
                continue
            sends = [torch.randint(0, 256, (in_bytes,), dtype=torch.uint8, device="cuda") for _ in range(n)]
            recvs = [torch.empty(n * s, dtype=torch.uint8, device="cuda") for _ in range(n)]
            for impl in impls:
                in_place = impl.endswith("swap")
                if in_place:
                    work = [t.clone() if t.numel() == n * s else None for t in sends]
                    rb = work
                else:
                    work, rb = sends, recvs
                # the inputs (and clones) are written on torch's stream; the
                # collective runs on `stream` (the caller orders them, as with
                # NCCL): without this a 2 GiB randint can still be running
                torch.cuda.synchronize()
                fn = cc.all_gather if kind == "allgather" else cc.all_to_all
                plan = None
                if args.api == "plan":
                    plan = cc.Plan(comms, kind, work, rb, s, impl=impl)

                    def call():
                        plan.launch(stream)
                else:
                    def call():
                        fn(comms, work, rb, s, impl=impl, streams=stream)

                with torch.cuda.stream(stream):
                    for _ in range(3):
                        call()
                stream.synchronize()
                # parity of every chunk of every rank (device compare); the
                # in-place swap is checked against the untouched inputs
                parity = True
                out = work if in_place else recvs
                for i in range(n):
                    for j in range(n):
                        src = sends[i][:s] if kind == "allgather" else sends[i][j * s:(j + 1) * s]
                        parity &= bool(torch.equal(out[j][i * s:(i + 1) * s], src))
                iters = int(max(5, min(500, 4e9 / (2 * n * n * s))))
                c0 = comms[0].counters()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                host = 0.0
                e0.record(stream)
                for _ in range(iters):
                    t0 = time.perf_counter()
                    call()
                    host += time.perf_counter() - t0
                e1.record(stream)
                stream.synchronize()
                c1 = comms[0].counters()
                total_ms = e0.elapsed_time(e1) / iters
                iso = []
                for _ in range(5):
                    stream.synchronize()
                    e0.record(stream)
                    call()
                    e1.record(stream)
                    stream.synchronize()
                    iso.append(e0.elapsed_time(e1))
                iso.sort()
                # Phase attribution from one traced, isolated collective of the
                # same plan (recorded plans trace their replayed graph).
                stream.synchronize()
                with cc.Trace(comms[0]) as tr:
                    call()
                    stream.synchronize()
                phases, traced_ns = trace_phases(tr.events)
                if plan is not None:
                    plan.destroy()
                torch.cuda.synchronize()
                bw = busbw(n, s, total_ms / 1e3)
                hbm = alg_hbm_bytes(kind, impl, s, n) / (total_ms / 1e3) / 1e9
                total_ns = total_ms * 1e6
                ph = {k: "" for k in ("control", "schedule", "copy", "sync", "trigger")}
                if phases and traced_ns > 0:  # fractions of the traced path, applied to total_ns
                    ph = {k: round(v / traced_ns * total_ns) for k, v in phases.items()}
                rows.append({
                    "impl": impl, "api": args.api, "collective": kind, "gpus": 1, "size_bytes": s,
                    "total_ns": round(total_ns), "control_ns": ph["control"], "schedule_ns": ph["schedule"],
                    "copy_ns": ph["copy"], "sync_ns": ph["sync"], "trigger_ns": ph["trigger"], "ranks": n,
                    "host_ns": round(host / iters * 1e9), "traced_ns": round(traced_ns),
                    "isolated_ns": round(iso[len(iso) // 2] * 1e6), "busbw_gbs": round(bw, 3),
                    "hbm_gbs": round(hbm, 1), "roofline_frac": round(hbm / peak, 4),
                    "api_calls": round((c1["api_calls"] - c0["api_calls"]) / iters, 1),
                    "kernels": round((c1["kernels"] - c0["kernels"]) / iters, 2),
                    "graphs": round((c1["graph_launches"] - c0["graph_launches"]) / iters, 2),
                    "parity": parity,
                })
                print(",".join(str(rows[-1][c]) for c in SWEEP_COLUMNS), flush=True)
            del sends, recvs
            torch.cuda.empty_cache()
    # CPU reference at the small sizes (the reference's compile() + byte executor).
    cpu_rows = []
    for kind in ("allgather", "alltoall"):
        for s in sizes[:6]:
            dt, label, cores, _ = cpu_reference_step(kind, n, s)
            cpu_rows.append({"impl": f"cpu_{label}", "collective": kind, "gpus": 0, "size_bytes": s,
                             "total_ns": round(dt * 1e9), "ranks": n, "busbw_gbs": round(busbw(n, s, dt), 3)})
    with open(out_path, "w") as f:
        f.write(",".join(SWEEP_COLUMNS) + "\n")
        for r in rows + cpu_rows:
            f.write(",".join(str(r.get(c, "")) for c in SWEEP_COLUMNS) + "\n")
    # winner grid (winner_grid, sweep.cpp:186-218)
    best = {}
    for r in rows:
        key = (r["collective"], r["size_bytes"])
        if key not in best or r["total_ns"] < best[key]["total_ns"]:
            best[key] = r
    for (kind, s), r in sorted(best.items()):
        print(f"winner {kind} s={s}: {r['impl']} {r['total_ns']} ns", flush=True)
    cc.destroy_all(comms)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--algo", default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-energy", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=40, help="timed steps of the end-to-end leg (at least --steps)")
    ap.add_argument("--sweep", action="store_true", help="size sweep of every implementation (CSV)")
    ap.add_argument("--ranks", type=int, default=NRANKS)
    ap.add_argument("--sweep-out", default=os.path.join(ROOT, "gpurun_out", "sweep.csv"))
    ap.add_argument("--max-bytes", type=float, default=96e9)
    ap.add_argument("--sweep-impls", default="", help="comma list: only these implementations")
    ap.add_argument("--sweep-kinds", default="", help="comma list: allgather,alltoall")
    ap.add_argument("--sweep-sizes", default="", help="comma list of per-peer chunk bytes")
    ap.add_argument("--api", default="eager", choices=["eager", "plan"],
                    help="sweep through the collective calls or through explicit plans")
    ap.add_argument("--interference", action="store_true", help="C4: all-gather beside a bf16 GEMM")
    ap.add_argument("--interference-chunk", type=int, default=256 << 20)
    ap.add_argument("--interference-impls", default="sm,sm@16,sm@32,sm@64,pcpy,b2b,pcpy:host,b2b:host,sm:host")
    ap.add_argument("--interference-host-chunk", type=int, default=16 << 20)
    ap.add_argument("--interference-out", default=os.path.join(ROOT, "gpurun_out", "interference.json"))
    ap.add_argument("--gemm-iters", type=int, default=200)
    ap.add_argument("--gemm-priority", default="same", choices=["same", "high"])
    ap.add_argument("--sync-chain", action="store_true", help="producer GEMM -> all-gather chain overhead")
    ap.add_argument("--sync-gemm", type=int, default=4096)
    ap.add_argument("--sync-out", default=os.path.join(ROOT, "gpurun_out", "sync_chain.json"))
    ap.add_argument("--sweep-rs", action="store_true", help="reduce-scatter sweep (bf16 sum)")
    # torchrun (N > 1) only: see bench_mgpu.py
    ap.add_argument("--no-nccl", action="store_true", help="skip the NCCL comparator")
    ap.add_argument("--no-mgpu-sweep", action="store_true", help="skip the one-rank-per-GPU size sweep")
    ap.add_argument("--mgpu-sweep-max", type=float, default=float(1 << 30), help="largest sweep chunk (bytes)")
    ap.add_argument("--mgpu-budget", type=float, default=240.0, help="no new sweep size after this many s")
    ap.add_argument("--mgpu-deadline", type=float, default=600.0, help="watchdog: print and exit after this many s")
    ap.add_argument("--mgpu-verbose", action="store_true")
    ap.add_argument("--no-mgpu-experiments", action="store_true", help="skip the multi-GPU design experiments")
    ap.add_argument("--no-mgpu-interference", action="store_true", help="skip the multi-GPU GEMM interference phase")
    args = ap.parse_args()
    if args.sweep_rs:
        run_sweep_rs(args)
    elif args.sync_chain:
        run_sync_chain(args)
    elif args.interference:
        run_interference(args)
    elif args.sweep:
        run_sweep(args)
    elif args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
