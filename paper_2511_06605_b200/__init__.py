"""cecoll — B200-native copy-engine collectives (Python host layer).

Thin ctypes bindings over the C ABI in include/cecoll.h (libcecoll.so, built
in-tree by build()). The vocabulary is the reference's: collective kinds
allgather/alltoall, implementations pcpy/bcst/swap/b2b/prelaunch_* (plus the
B200 SM path "sm"), per-peer chunk size s, and the rank/chunk layout of
proj/src/compiler.cpp:115-126.

The product path is libcecoll.so only: if it is missing every entry point
raises; nothing here falls back to a CPU or torch implementation.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Callable, Sequence

# Streams that wait on flags must not share a hardware queue with the stream
# that writes them; give the driver its maximum number of queues. Must be set
# before the CUDA context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcecoll.so")
CSRC = os.path.join(HERE, "csrc")

ALLGATHER, ALLTOALL = 0, 1
KINDS = {"allgather": ALLGATHER, "ag": ALLGATHER, "alltoall": ALLTOALL, "aa": ALLTOALL}
IMPLS = {
    "auto": -1,
    "pcpy": 0,
    "baseline": 0,
    "bcst": 1,
    "swap": 2,
    "b2b": 3,
    "prelaunch_pcpy": 4,
    "prelaunch_bcst": 5,
    "prelaunch_swap": 6,
    "prelaunch_b2b": 7,
    "sm": 8,
    "hybrid": 9,
    "pull": 10,
}
IMPL_NAMES = {v: k for k, v in IMPLS.items() if k != "baseline"}
# implementations_for (compiler.cpp:77-85) + the SM path
IMPLS_FOR = {
    "allgather": ["pcpy", "bcst", "b2b", "prelaunch_pcpy", "prelaunch_bcst", "prelaunch_b2b"],
    "alltoall": ["pcpy", "swap", "b2b", "prelaunch_pcpy", "prelaunch_swap", "prelaunch_b2b"],
}
STATUS = {
    0: "success",
    1: "invalid argument",
    2: "unsupported",
    3: "CUDA error",
    4: "timeout",
    5: "no CUDA device",
    6: "buffer not registered",
    7: "internal error",
}
DEFAULT_LANES = 16  # engines_per_gpu default of the reference topology (topology.hpp:34)


class CecollError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"cecoll: {STATUS.get(status, status)}: {what}")


class InvalidArgument(CecollError, ValueError):
    pass


def build(force: bool = False) -> str:
    """Compile libcecoll.so for sm_100a in-tree (nvcc cross-compiles without a GPU)."""
    cmd = ["make", "-s", "-C", CSRC, "-j8"]
    if force:
        subprocess.run(["make", "-s", "-C", CSRC, "clean"], check=True)
    subprocess.run(cmd, check=True)
    return LIB_PATH


class ModelParams(C.Structure):
    """cecoll_model_t (include/cecoll.h): the B200 cost model's parameters."""
    _fields_ = [(k, C.c_double) for k in ("t_kernel", "t_graph", "t_branch", "t_node", "t_trigger", "bw_copy",
                                          "bw_fan", "bw_ce", "bw_lanes", "bw_swap", "l2_boost", "l2_bytes",
                                          "folded_max_bytes",
                                          "prelaunch_gain_threshold", "t_stream", "stream_min_bytes",
                                          "l2_boost_swap")]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


def lib():
    """The loaded libcecoll.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libcecoll.so not built ({LIB_PATH}); run paper_2511_06605_b200.build()")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, sz = C.c_void_p, C.c_int, C.c_int64, C.c_size_t
    sig = {
        "cecoll_strerror": ([i32], C.c_char_p),
        "cecoll_impl_name": ([i32], C.c_char_p),
        "cecoll_parse_impl": ([C.c_char_p], i32),
        "cecoll_impl_valid_for": ([i32, i32], i32),
        "cecoll_last_error": ([], C.c_char_p),
        "cecoll_program_compile": ([i32, i32, i64, i32, i32, C.POINTER(vp)], i32),
        "cecoll_program_dump": ([vp, C.c_char_p, sz], i64),
        "cecoll_program_metrics": ([vp, C.POINTER(i64)], i32),
        "cecoll_program_traffic": ([vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)], i32),
        "cecoll_program_validate": ([vp, i32], i32),
        "cecoll_program_free": ([vp], None),
        "cecoll_program_parse": ([C.c_char_p, i32, i64, i32, C.POINTER(vp)], i32),
        "cecoll_plan_create_program": ([C.POINTER(vp), i32, vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)], i32),
        "cecoll_reference_select": ([i32, i64], i32),
        "cecoll_select": ([i32, i64, i32, i32], i32),
        "cecoll_comm_init_all": ([C.POINTER(vp), i32, C.POINTER(i32)], i32),
        "cecoll_comm_init_rank": ([C.POINTER(vp), i32, i32, i32, EXCHANGE_FN, vp], i32),
        "cecoll_comm_init_ranks": ([C.POINTER(vp), i32, i32, i32, i32, EXCHANGE_FN, vp], i32),
        "cecoll_exchange_check": ([i32, i32, i32, i32, EXCHANGE_FN, vp, C.POINTER(C.c_int32)], i32),
        "cecoll_comm_destroy": ([vp], i32),
        "cecoll_comm_info": ([vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)], i32),
        "cecoll_register": ([vp, vp, sz], i32),
        "cecoll_deregister": ([vp, vp], i32),
        "cecoll_mem_alloc": ([vp, sz, C.POINTER(vp)], i32),
        "cecoll_mem_free": ([vp, vp], i32),
        "cecoll_trace_begin": ([vp], i32),
        "cecoll_trace_end": ([vp, C.c_char_p, sz, C.POINTER(sz)], i32),
        "cecoll_allgather": ([vp, vp, sz, i32, vp, vp], i32),
        "cecoll_alltoall": ([vp, vp, sz, i32, vp, vp], i32),
        "cecoll_group_start": ([], i32),
        "cecoll_group_end": ([], i32),
        "cecoll_collective_n": ([i32, C.POINTER(vp), i32, C.POINTER(vp), C.POINTER(vp), sz, i32, C.POINTER(vp)], i32),
        "cecoll_reduce_scatter": ([vp, vp, sz, i32, i32, i32, vp, vp], i32),
        "cecoll_reduce_scatter_n": ([C.POINTER(vp), i32, C.POINTER(vp), C.POINTER(vp), sz, i32, i32, i32,
                                     C.POINTER(vp)], i32),
        "cecoll_plan_create": ([C.POINTER(vp), i32, i32, C.POINTER(vp), C.POINTER(vp), sz, i32, C.POINTER(vp)], i32),
        "cecoll_plan_launch": ([vp, C.POINTER(vp)], i32),
        "cecoll_plan_destroy": ([vp], i32),
        "cecoll_plan_disarm": ([vp], i32),
        "cecoll_plan_arm": ([vp], i32),
        "cecoll_comm_get_async_error": ([vp, C.POINTER(i32)], i32),
        "cecoll_plan_trigger": ([vp, C.POINTER(vp)], i32),
        "cecoll_comm_counters": ([vp, C.POINTER(i64)], i32),
        "cecoll_mc_window_create": ([vp, sz, C.POINTER(vp), C.POINTER(vp)], i32),
        "cecoll_mc_allgather": ([vp, vp, sz, vp], i32),
        "cecoll_mc_handle_type": ([vp], C.c_char_p),
        "cecoll_mc_window_destroy": ([vp], i32),
        "cecoll_plan_info": ([vp, C.c_char_p, sz, C.POINTER(sz)], i32),
        "cecoll_comm_last_plan_info": ([vp, C.c_char_p, sz, C.POINTER(sz)], i32),
        "cecoll_comm_set_sm_budget": ([vp, i32], i32),
        "cecoll_tune": ([C.POINTER(vp), i32, i64, C.POINTER(vp)], i32),
        "cecoll_tune_table": ([vp, C.c_char_p, sz, C.POINTER(sz)], i32),
        "cecoll_tune_load": ([vp, C.c_char_p], i32),
        "cecoll_tune_report": ([vp, C.c_char_p, sz, C.POINTER(sz)], i32),
        "cecoll_select_budget": ([i32, i64, i32, i32, i32], i32),
        "cecoll_model_default": ([C.POINTER(ModelParams)], None),
        "cecoll_model_predict": ([C.POINTER(ModelParams), i32, i32, i64, i32, C.POINTER(C.c_double)], i32),
        "cecoll_model_winner": ([C.POINTER(ModelParams), i32, i64, i32], i32),
        "cecoll_model_fit": ([C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(i64), C.POINTER(C.c_int),
                              C.POINTER(C.c_double), i32, C.c_uint64, i32, C.POINTER(ModelParams),
                              C.POINTER(C.c_double), C.c_char_p, sz], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


EXPORTED_SYMBOLS = [
    "cecoll_strerror", "cecoll_impl_name", "cecoll_parse_impl", "cecoll_impl_valid_for", "cecoll_last_error",
    "cecoll_program_compile", "cecoll_program_dump", "cecoll_program_metrics", "cecoll_program_traffic",
    "cecoll_program_validate", "cecoll_program_free", "cecoll_reference_select", "cecoll_select",
    "cecoll_comm_init_all", "cecoll_comm_init_rank", "cecoll_comm_destroy", "cecoll_comm_info",
    "cecoll_register", "cecoll_deregister", "cecoll_allgather", "cecoll_alltoall", "cecoll_group_start",
    "cecoll_group_end", "cecoll_plan_create", "cecoll_plan_launch", "cecoll_plan_destroy", "cecoll_comm_counters",
    "cecoll_program_parse", "cecoll_plan_create_program", "cecoll_comm_init_ranks", "cecoll_exchange_check",
    "cecoll_collective_n", "cecoll_plan_disarm", "cecoll_plan_arm", "cecoll_plan_trigger",
    "cecoll_comm_get_async_error", "cecoll_reduce_scatter", "cecoll_reduce_scatter_n",
    "cecoll_mem_alloc", "cecoll_mem_free", "cecoll_trace_begin", "cecoll_trace_end",
    "cecoll_mc_window_create", "cecoll_mc_allgather", "cecoll_mc_handle_type", "cecoll_mc_window_destroy",
    "cecoll_plan_info", "cecoll_comm_last_plan_info", "cecoll_comm_set_sm_budget", "cecoll_select_budget",
    "cecoll_model_default", "cecoll_model_predict", "cecoll_model_winner", "cecoll_model_fit",
    "cecoll_tune", "cecoll_tune_table", "cecoll_tune_load", "cecoll_tune_report",
]
DTYPES = {"f32": 0, "float32": 0, "bf16": 1, "bfloat16": 1, "f16": 2, "float16": 2}
REDOPS = {"sum": 0, "max": 1, "min": 2}


def _check(status: int, what: str = ""):
    if status != 0:
        msg = lib().cecoll_last_error().decode(errors="replace")
        cls = InvalidArgument if status in (1, 2) else CecollError
        raise cls(status, f"{what}: {msg}" if what else msg)


def _kind(kind) -> int:
    if isinstance(kind, int):
        return kind
    return KINDS[kind]


def _impl(impl) -> int:
    if isinstance(impl, int):
        return impl
    if impl not in IMPLS:
        raise InvalidArgument(1, f"unknown implementation {impl!r}")
    return IMPLS[impl]


def impl_name(impl: int) -> str:
    return lib().cecoll_impl_name(impl).decode()


# ---------------------------------------------------------------------------
# Command programs (CPU only) — compile() / dump_program() / static_metrics()
# / account_traffic() / validate_program() (proj/src/{compiler,program,verifier}.cpp)
# ---------------------------------------------------------------------------


class Program:
    """A compiled command program (≙ dmasim::CommandProgram)."""

    def __init__(self, kind, impl, chunk_bytes: int, nranks: int, lanes_per_rank: int = DEFAULT_LANES,
                 _handle=None):
        self.kind, self.impl, self.chunk, self.nranks = kind, impl, chunk_bytes, nranks
        if _handle is not None:
            self._h = _handle
            return
        h = C.c_void_p()
        _check(
            lib().cecoll_program_compile(_kind(kind), _impl(impl), chunk_bytes, nranks, lanes_per_rank, C.byref(h)),
            f"compile {kind}/{impl} s={chunk_bytes} n={nranks}",
        )
        self._h = h

    @classmethod
    def parse(cls, dump_text: str, kind, chunk_bytes: int, nranks: int) -> "Program":
        """Read the reference's dump_program text (e.g. `dmasim compile` output)."""
        h = C.c_void_p()
        _check(lib().cecoll_program_parse(dump_text.encode(), _kind(kind), chunk_bytes, nranks, C.byref(h)),
               "program_parse")
        return cls(kind, None, chunk_bytes, nranks, _handle=h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cecoll_program_free(self._h)
            self._h = None

    def dump(self) -> str:
        cap = 1 << 22
        buf = C.create_string_buffer(cap)
        k = lib().cecoll_program_dump(self._h, buf, cap)
        if k < 0:
            raise CecollError(7, "dump buffer too small")
        return buf.raw[:k].decode()

    def metrics(self) -> dict:
        out = (C.c_int64 * 5)()
        _check(lib().cecoll_program_metrics(self._h, out))
        return dict(zip(["data_commands", "sync_commands", "poll_commands", "engines_used", "doorbells"], list(out)))

    def traffic(self) -> dict:
        t = (C.c_int64 * 3)()
        rr = (C.c_int64 * self.nranks)()
        rw = (C.c_int64 * self.nranks)()
        _check(lib().cecoll_program_traffic(self._h, t, rr, rw))
        return {"read": t[0], "write": t[1], "link": t[2], "rank_read": list(rr), "rank_write": list(rw)}

    def validate(self, lanes_per_rank: int = DEFAULT_LANES) -> str | None:
        st = lib().cecoll_program_validate(self._h, lanes_per_rank)
        return None if st == 0 else lib().cecoll_last_error().decode()


def reference_select(kind, chunk_bytes: int) -> str | None:
    """select_implementation (compiler.cpp:305-318): the reference's MI300X table."""
    r = lib().cecoll_reference_select(_kind(kind), chunk_bytes)
    return None if r < -1 else IMPL_NAMES[r]


def select(kind, chunk_bytes: int, nranks: int, ndevices: int, sm_budget: int = 0) -> str:
    """The B200 selector (measured thresholds); with an SM budget it prefers
    the copy engines across devices (cecoll_select_budget)."""
    if sm_budget:
        return IMPL_NAMES[lib().cecoll_select_budget(_kind(kind), chunk_bytes, nranks, ndevices, sm_budget)]
    return IMPL_NAMES[lib().cecoll_select(_kind(kind), chunk_bytes, nranks, ndevices)]


class Model:
    """The B200 cost model (csrc/model.cpp): predict the device
    time of a collective, pick the winner at a size, fit to measurements with
    the reference's calibrate() procedure. CPU only."""

    def __init__(self, params: dict | None = None):
        self.p = ModelParams()
        lib().cecoll_model_default(C.byref(self.p))
        for k, v in (params or {}).items():
            setattr(self.p, k, float(v))

    def predict_ns(self, kind, impl, chunk_bytes: int, nranks: int) -> float:
        out = C.c_double()
        _check(lib().cecoll_model_predict(C.byref(self.p), _kind(kind), _impl(impl), chunk_bytes, nranks,
                                          C.byref(out)), "model_predict")
        return out.value

    def winner(self, kind, chunk_bytes: int, nranks: int) -> str:
        return IMPL_NAMES[lib().cecoll_model_winner(C.byref(self.p), _kind(kind), chunk_bytes, nranks)]

    @classmethod
    def fit(cls, rows, seed: int = 0, iterations: int = 2000):
        """rows: (kind, impl, chunk_bytes, nranks, ns). Returns (model, residual, report)."""
        k = len(rows)
        kinds = (C.c_int * k)(*[_kind(r[0]) for r in rows])
        impls = (C.c_int * k)(*[_impl(r[1]) for r in rows])
        sizes = (C.c_int64 * k)(*[int(r[2]) for r in rows])
        ns_ = (C.c_int * k)(*[int(r[3]) for r in rows])
        times = (C.c_double * k)(*[float(r[4]) for r in rows])
        m = cls()
        res = C.c_double()
        rep = C.create_string_buffer(1 << 16)
        _check(lib().cecoll_model_fit(kinds, impls, sizes, ns_, times, k, seed, iterations, C.byref(m.p),
                                      C.byref(res), rep, len(rep)), "model_fit")
        return m, res.value, rep.value.decode()


def _json_out(fn, handle) -> dict:
    import json

    n = C.c_size_t()
    _check(fn(handle, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(fn(handle, buf, n.value + 1, C.byref(n)))
    return json.loads(buf.value.decode())


# ---------------------------------------------------------------------------
# Communicators and collectives
# ---------------------------------------------------------------------------


def _ptr(x) -> int:
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    raise TypeError(f"expected a device pointer or tensor, got {type(x)}")


def _stream(s) -> int | None:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream  # torch.cuda.Stream


class Comm:
    """One rank of a communicator (≙ ncclComm_t)."""

    def __init__(self, handle, owner=None):
        self._h = handle
        self._owner = owner  # keeps the exchange callback alive (multi-process)
        r, n, d = C.c_int(), C.c_int(), C.c_int()
        _check(lib().cecoll_comm_info(self._h, C.byref(r), C.byref(n), C.byref(d)))
        self.rank, self.nranks, self.device = r.value, n.value, d.value

    @staticmethod
    def init_all(devices: Sequence[int]) -> list["Comm"]:
        """Single process driving every rank (devices may repeat: co-resident ranks)."""
        n = len(devices)
        hs = (C.c_void_p * n)()
        devs = (C.c_int * n)(*devices)
        _check(lib().cecoll_comm_init_all(hs, n, devs), "comm_init_all")
        return [Comm(C.c_void_p(hs[i])) for i in range(n)]

    @staticmethod
    def init_rank(nranks: int, rank: int, device: int, exchange: Callable[[bytes], list[bytes]]) -> "Comm":
        """One rank per process; `exchange(mine) -> [bytes of every process]` is an all-gather."""
        return Comm.init_ranks(nranks, rank, 1, device, exchange)[0]

    @staticmethod
    def init_ranks(nranks: int, first: int, nlocal: int, device: int,
                   exchange: Callable[[bytes], list[bytes]]) -> list["Comm"]:
        """This process owns ranks [first, first+nlocal) on `device` (co-resident)."""
        cb = _make_exchange(exchange, nranks // nlocal)
        hs = (C.c_void_p * nlocal)()
        _check(lib().cecoll_comm_init_ranks(hs, nranks, first, nlocal, device, cb, None), "comm_init_ranks")
        return [Comm(C.c_void_p(hs[k]), owner=cb) for k in range(nlocal)]

    def register(self, buf, nbytes: int | None = None):
        """Collective in multi-process communicators (symmetric windows)."""
        ptr = _ptr(buf)
        if nbytes is None:
            nbytes = buf.numel() * buf.element_size()
        _check(lib().cecoll_register(self._h, ptr, nbytes), "register")

    def deregister(self, buf):
        _check(lib().cecoll_deregister(self._h, _ptr(buf)), "deregister")

    def mem_alloc(self, nbytes: int):
        """Library-owned, registered device buffer of `nbytes` (rounded up to
        2 MiB pages; collective in multi-process communicators). Returned as a
        uint8 CUDA tensor that does not own the memory: release it with
        mem_free."""
        import torch

        p = C.c_void_p()
        _check(lib().cecoll_mem_alloc(self._h, nbytes, C.byref(p)), "mem_alloc")

        class _View:  # __cuda_array_interface__ lets torch wrap the pointer without a copy
            __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (p.value, False),
                                        "version": 3, "strides": None}

        with torch.cuda.device(self.device):
            return torch.as_tensor(_View(), device=f"cuda:{self.device}")

    def mem_free(self, buf):
        _check(lib().cecoll_mem_free(self._h, _ptr(buf)), "mem_free")

    def set_sm_budget(self, max_ctas: int):
        """Plans created from now on in this world launch at most `max_ctas`
        CTAs per kernel (0: full grid); AUTO prefers the copy engines."""
        _check(lib().cecoll_comm_set_sm_budget(self._h, max_ctas), "comm_set_sm_budget")

    def tuned_table(self) -> list:
        """cecoll_tune_table: the world's measured winner grid as
        [(kind, chunk_bytes, impl), ...] (empty: the static selector)."""
        n = C.c_size_t()
        _check(lib().cecoll_tune_table(self._h, None, 0, C.byref(n)), "tune_table")
        buf = C.create_string_buffer(n.value)
        _check(lib().cecoll_tune_table(self._h, buf, n.value, C.byref(n)), "tune_table")
        rows = []
        for line in buf.value.decode().splitlines():
            kind, s, impl = line.split()
            rows.append((kind, int(s), impl))
        return rows

    def tune_report(self) -> dict:
        """cecoll_tune_report: {(kind, chunk_bytes): {"us": {impl: µs}, "winner": impl}}."""
        n = C.c_size_t()
        _check(lib().cecoll_tune_report(self._h, None, 0, C.byref(n)), "tune_report")
        buf = C.create_string_buffer(n.value)
        _check(lib().cecoll_tune_report(self._h, buf, n.value, C.byref(n)), "tune_report")
        out = {}
        for line in buf.value.decode().splitlines():
            head, win = line.split(" -> ")
            parts = head.split()
            us = {k: float(v) for k, v in (p.split("=") for p in parts[2:])}
            out[(parts[0], int(parts[1]))] = {"us": us, "winner": win}
        return out

    def load_tuned(self, rows):
        """cecoll_tune_load: install a table ([(kind, chunk_bytes, impl)] or
        its text form); an empty one clears it."""
        text = rows if isinstance(rows, str) else "".join(f"{k} {s} {i}\n" for k, s, i in rows)
        _check(lib().cecoll_tune_load(self._h, text.encode()), "tune_load")

    def last_plan_info(self) -> dict:
        """cecoll_comm_last_plan_info: what the latest eager collective ran."""
        return _json_out(lib().cecoll_comm_last_plan_info, self._h)

    def counters(self) -> dict:
        out = (C.c_int64 * 8)()
        _check(lib().cecoll_comm_counters(self._h, out))
        # graph_launches: prelaunch graphs (their kernels are not in `kernels`);
        # recorded_launches: replays of a recorded command list (their kernels,
        # copies and flag operations are counted in the other keys).
        keys = ["collectives", "copies", "flag_writes", "flag_waits", "kernels", "graph_launches", "api_calls",
                "recorded_launches"]
        return dict(zip(keys, list(out)))

    def async_error(self):
        """None, or the CecollError a device-side poll of this world recorded
        (CECOLL_TIMEOUT after 20 s without the peer's signal)."""
        code = C.c_int32(0)
        _check(lib().cecoll_comm_get_async_error(self._h, C.byref(code)), "comm_get_async_error")
        if code.value == 0:
            return None
        return CecollError(code.value, lib().cecoll_last_error().decode(errors="replace"))

    def destroy(self):
        if self._h is not None:
            h, self._h = self._h, None
            _check(lib().cecoll_comm_destroy(h), "comm_destroy")


class McWindow:
    """EXPERIMENTAL NVLS (switch multicast) all-gather window (include/cecoll.h,
    csrc/mcast.cpp). Collective to create (one process per GPU); `recv` is this
    rank's window: after allgather(send, s) it holds rank i's chunk at
    [i*s, (i+1)*s). Raises CecollError (unsupported) where the node offers no
    multicast objects."""

    def __init__(self, comm: "Comm", chunk_capacity: int):
        import torch

        h, p = C.c_void_p(), C.c_void_p()
        _check(lib().cecoll_mc_window_create(comm._h, chunk_capacity, C.byref(h), C.byref(p)), "mc_window_create")
        self._h = h
        self.capacity = chunk_capacity
        self.handle_type = lib().cecoll_mc_handle_type(h).decode()
        nbytes = comm.nranks * chunk_capacity

        class _View:
            __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (p.value, False),
                                        "version": 3, "strides": None}

        with torch.cuda.device(comm.device):
            self.recv = torch.as_tensor(_View(), device=f"cuda:{comm.device}")

    def allgather(self, send, chunk_bytes: int, stream=None):
        _check(lib().cecoll_mc_allgather(self._h, _ptr(send), chunk_bytes, _stream(stream)), "mc_allgather")

    def destroy(self):
        if self._h is not None:
            _check(lib().cecoll_mc_window_destroy(self._h), "mc_window_destroy")
            self._h = None


class Trace:
    """Records the hardware timeline of every collective issued inside the
    block, in the reference's trace-event format (sim.cpp:523-544): after the
    block, `events` is the list of {"name", "ph", "ts", "pid", "tid"} dicts
    (chrome://tracing / Perfetto load `save(path)` directly).

        with cc.Trace(comms[0]) as t:
            cc.all_to_all(comms, sends, recvs, s, impl="pcpy")
        t.save("aa_pcpy.json")
    """

    def __init__(self, comm: Comm):
        self._comm = comm
        self.events: list[dict] = []

    def __enter__(self):
        _check(lib().cecoll_trace_begin(self._comm._h), "trace_begin")
        return self

    def __exit__(self, *exc):
        n = C.c_size_t()
        _check(lib().cecoll_trace_end(self._comm._h, None, 0, C.byref(n)), "trace_end")
        buf = C.create_string_buffer(n.value + 1)
        _check(lib().cecoll_trace_end(self._comm._h, buf, n.value + 1, C.byref(n)), "trace_end")
        import json

        self.events = json.loads(buf.value.decode())
        return False

    def save(self, path: str):
        import json

        with open(path, "w") as f:
            json.dump(self.events, f, indent=1)


def tune(comms: Sequence[Comm], max_chunk: int = 64 << 20, streams=None):
    """cecoll_tune: measure every applicable implementation on this machine
    (4 KiB x 4^k chunks up to max_chunk) and let AUTO use the winners. Pass
    every local communicator of the world (every process calls it)."""
    n = len(comms)
    hs = (C.c_void_p * n)(*[c._h for c in comms])
    ss = None
    if streams is not None:
        if not isinstance(streams, (list, tuple)):
            streams = [streams] * n
        ss = (C.c_void_p * n)(*[_stream(s) for s in streams])
    _check(lib().cecoll_tune(hs, n, max_chunk, ss), "tune")


def destroy_all(comms: Sequence[Comm]):
    for c in comms:
        c.destroy()


def _make_exchange(exchange, nprocs):
    def _cb(ctx, mine, nbytes, out):
        try:
            data = C.string_at(mine, nbytes)
            parts = exchange(data)
            if len(parts) != nprocs or any(len(p) != nbytes for p in parts):
                return 1
            blob = b"".join(parts)
            C.memmove(out, blob, len(blob))
            return 0
        except Exception:  # noqa: BLE001 - reported as a status code across the ABI
            return 1

    return EXCHANGE_FN(_cb)


def exchange_check(nranks: int, first: int, nlocal: int, device: int, exchange) -> list[int]:
    """Run only the init exchange (host, no CUDA): every rank's device."""
    cb = _make_exchange(exchange, nranks // nlocal)
    out = (C.c_int32 * nranks)()
    _check(lib().cecoll_exchange_check(nranks, first, nlocal, device, cb, None, out), "exchange_check")
    return list(out)


def torch_exchange(group=None):
    """An exchange callback over torch.distributed (gloo or nccl object collectives)."""
    import torch.distributed as dist

    def ex(mine: bytes) -> list[bytes]:
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, mine, group=group)
        return out

    return ex


def _collective(kind, comms, sends, recvs, chunk_bytes, impl, streams):
    """The n per-rank calls of one group as a single C call (cecoll_collective_n)."""
    if isinstance(comms, Comm):
        comms, sends, recvs = [comms], [sends], [recvs]
        streams = [streams] if not isinstance(streams, (list, tuple)) else streams
    n = len(comms)
    if streams is None or not isinstance(streams, (list, tuple)):
        streams = [streams] * n
    arr = C.c_void_p * n
    _check(lib().cecoll_collective_n(kind, arr(*[c._h.value for c in comms]), n, arr(*[_ptr(s) for s in sends]),
                                     arr(*[_ptr(r) for r in recvs]), chunk_bytes, _impl(impl),
                                     arr(*[_stream(st) for st in streams])),
           "allgather" if kind == ALLGATHER else "alltoall")


def all_gather(comms, sends, recvs, chunk_bytes: int, impl="auto", streams=None):
    """recv[r] (n*s bytes) gets rank i's s-byte chunk at [i*s, (i+1)*s) (compiler.cpp:115-122)."""
    _collective(ALLGATHER, comms, sends, recvs, chunk_bytes, impl, streams)


def all_to_all(comms, sends, recvs, chunk_bytes: int, impl="auto", streams=None):
    """send[r] chunk j (s bytes) lands in recv[j] slot r (compiler.cpp:124-126, 156-157)."""
    _collective(ALLTOALL, comms, sends, recvs, chunk_bytes, impl, streams)


def _dtype(dtype) -> int:
    if isinstance(dtype, int):
        return dtype
    name = str(dtype).replace("torch.", "")
    if name not in DTYPES:
        raise InvalidArgument(1, f"unsupported reduce-scatter dtype {dtype!r}")
    return DTYPES[name]


def reduce_scatter(comms, sends, recvs, count: int, dtype="bf16", op="sum", impl="auto", streams=None):
    """recv[j] (count elements) = op over ranks i, in rank order, of send[i][j*count:(j+1)*count]
    (fp32 accumulation, one round-to-nearest-even)."""
    if isinstance(comms, Comm):
        comms, sends, recvs = [comms], [sends], [recvs]
        streams = [streams] if not isinstance(streams, (list, tuple)) else streams
    n = len(comms)
    if streams is None or not isinstance(streams, (list, tuple)):
        streams = [streams] * n
    arr = C.c_void_p * n
    _check(lib().cecoll_reduce_scatter_n(arr(*[c._h.value for c in comms]), n, arr(*[_ptr(s) for s in sends]),
                                         arr(*[_ptr(r) for r in recvs]), count, _dtype(dtype), REDOPS[op],
                                         _impl(impl), arr(*[_stream(st) for st in streams])), "reduce_scatter")


class Plan:
    """A prelaunched plan: recorded once, armed ahead, triggered per launch."""

    def __init__(self, comms, kind, sends, recvs, chunk_bytes: int = 0, impl="prelaunch_pcpy",
                 program: Program | None = None):
        n = len(comms)
        hs = (C.c_void_p * n)(*[c._h.value for c in comms])
        ss = (C.c_void_p * n)(*[_ptr(x) for x in sends])
        rs = (C.c_void_p * n)(*[_ptr(x) for x in recvs])
        self._keep = (sends, recvs, program)  # buffers must outlive an armed plan
        self._n = n
        h = C.c_void_p()
        if program is not None:
            _check(lib().cecoll_plan_create_program(hs, n, program._h, ss, rs, C.byref(h)), "plan_create_program")
        else:
            _check(lib().cecoll_plan_create(hs, n, _kind(kind), ss, rs, chunk_bytes, _impl(impl), C.byref(h)),
                   "plan_create")
        self._h = h

    def _streams(self, streams):
        # The marshalled stream array is cached per streams argument: a plan is
        # relaunched with the same streams in latency-bound loops.
        key = tuple(streams) if isinstance(streams, (list, tuple)) else streams
        cache = self.__dict__.setdefault("_arrs", {})
        arr = cache.get(key)
        if arr is None:
            seq = list(streams) if isinstance(streams, (list, tuple)) else [streams] * self._n
            arr = cache[key] = (C.c_void_p * self._n)(*[_stream(s) for s in seq])
        return arr

    def launch(self, streams=None):
        st = _lib.cecoll_plan_launch(self._h, self._streams(streams))
        if st:
            _check(st, "plan_launch")

    def arm(self):
        """Launch the gated instance now (prelaunch_* plans; no-op otherwise)."""
        _check(lib().cecoll_plan_arm(self._h), "plan_arm")

    def trigger(self, streams=None):
        """Open the armed instance (arming first if needed) without re-arming."""
        _check(lib().cecoll_plan_trigger(self._h, self._streams(streams)), "plan_trigger")

    def disarm(self):
        """Cancel the armed instance (needed before torch.cuda.synchronize())."""
        _check(lib().cecoll_plan_disarm(self._h), "plan_disarm")

    def info(self) -> dict:
        """cecoll_plan_info: graph fallback, recording, movers, flag paths."""
        return _json_out(lib().cecoll_plan_info, self._h)

    def destroy(self):
        if self._h is not None:
            _check(lib().cecoll_plan_destroy(self._h), "plan_destroy")
            self._h = None
