"""ctypes bindings for the oracle — TEST INFRASTRUCTURE ONLY.

`Oracle` wraps oracle/liboracle.so (the plain-C restatement, cecoll_oracle.c);
`Reference` wraps oracle/_ref/libdmasim_ref.so (the reference's own compiler
and verifier sources compiled in place, see oracle/Makefile). Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libdmasim_ref.so")

KINDS = {"allgather": 0, "alltoall": 1}
IMPLS = ["pcpy", "bcst", "swap", "b2b", "prelaunch_pcpy", "prelaunch_bcst", "prelaunch_swap", "prelaunch_b2b"]
# implementations_for (compiler.cpp:77-85): base variants first.
IMPLS_FOR = {
    "allgather": ["pcpy", "bcst", "b2b", "prelaunch_pcpy", "prelaunch_bcst", "prelaunch_b2b"],
    "alltoall": ["pcpy", "swap", "b2b", "prelaunch_pcpy", "prelaunch_swap", "prelaunch_b2b"],
}
VERDICTS = {0: "ok", 1: "mismatch", 2: "hazard", 3: "invalid"}

ORA_MAX_CMDS = 40
ORA_MAX_QUEUES = 1024


class OraRef(C.Structure):
    _fields_ = [("gpu", C.c_int), ("buffer", C.c_int), ("offset", C.c_int64), ("length", C.c_int64)]


class OraCmd(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("src", OraRef),
        ("dst", OraRef),
        ("dst2", OraRef),
        ("peer", OraRef),
        ("size", C.c_int64),
        ("signal_target", C.c_int),
        ("poll_slot", C.c_int),
        ("expected_value", C.c_uint64),
    ]


class OraQueue(C.Structure):
    _fields_ = [
        ("gpu", C.c_int),
        ("engine", C.c_int),
        ("doorbell_count", C.c_int),
        ("ncmds", C.c_int),
        ("cmds", OraCmd * ORA_MAX_CMDS),
    ]


class OraProgram(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("chunk_size", C.c_int64),
        ("gpu_count", C.c_int),
        ("in_place", C.c_int),
        ("impl", C.c_int),
        ("prelaunched", C.c_int),
        ("nqueues", C.c_int),
        ("queues", OraQueue * ORA_MAX_QUEUES),
    ]


def build_oracle() -> None:
    """Compile oracle/liboracle.so (and oracle/_ref when the reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def splitmix_pattern(nbytes: int, rank: int, seed: int = 0) -> np.ndarray:
    """u64 word w of rank r = splitmix64(seed ^ (r << 48) ^ w)."""
    words = (nbytes + 7) // 8
    with np.errstate(over="ignore"):
        x = np.arange(words, dtype=np.uint64) ^ np.uint64(seed ^ (rank << 48))
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x.view(np.uint8)[:nbytes].copy()


def _ptrs(bufs):
    arr = (C.POINTER(C.c_uint8) * len(bufs))()
    for i, b in enumerate(bufs):
        arr[i] = b.ctypes.data_as(C.POINTER(C.c_uint8))
    return arr


class Oracle:
    def __init__(self, path: str = LIB):
        if not os.path.exists(path):
            build_oracle()
        L = C.CDLL(path)
        self.L = L
        L.ora_program_new.restype = C.POINTER(OraProgram)
        L.ora_program_free.argtypes = [C.POINTER(OraProgram)]
        L.ora_compile.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int, C.POINTER(OraProgram)]
        L.ora_dump.argtypes = [C.POINTER(OraProgram), C.c_char_p, C.c_size_t]
        L.ora_dump.restype = C.c_int64
        L.ora_static_metrics.argtypes = [C.POINTER(OraProgram), C.POINTER(C.c_int * 5)]
        L.ora_traffic.argtypes = [C.POINTER(OraProgram)] + [C.POINTER(C.c_int64)] * 5
        L.ora_verify.argtypes = [C.POINTER(OraProgram), C.c_int, C.c_uint64]
        L.ora_select.argtypes = [C.c_int, C.c_int64]
        L.ora_fill_pattern.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_uint64]
        L.ora_execute.argtypes = [C.POINTER(OraProgram), C.c_void_p, C.c_void_p]
        L.ora_check.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.ora_check.restype = C.c_int64
        L.ora_reference_result.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
        L.ora_reduce_scatter.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
        L.ora_parse_impl.argtypes = [C.c_char_p]
        L.ora_impl_name.restype = C.c_char_p

    def compile(self, kind: str, impl: str, s: int, n: int, engines: int = 16):
        p = self.L.ora_program_new()
        rc = self.L.ora_compile(IMPLS.index(impl), KINDS[kind], s, n, engines, p)
        if rc != 0:
            self.L.ora_program_free(p)
            raise ValueError(f"oracle compile rejected {kind}/{impl} s={s} n={n}")
        return p

    def free(self, p):
        self.L.ora_program_free(p)

    def dump(self, p) -> str:
        cap = 1 << 22
        buf = C.create_string_buffer(cap)
        k = self.L.ora_dump(p, buf, cap)
        assert k >= 0
        return buf.raw[:k].decode()

    def metrics(self, p):
        out = (C.c_int * 5)()
        self.L.ora_static_metrics(p, C.byref(out))
        return list(out)

    def traffic(self, p, n):
        tr, tw, tl = C.c_int64(), C.c_int64(), C.c_int64()
        gr, gw = (C.c_int64 * n)(), (C.c_int64 * n)()
        self.L.ora_traffic(p, C.byref(tr), C.byref(tw), C.byref(tl), gr, gw)
        return [tr.value, tw.value, tl.value], list(gr), list(gw)

    def verify(self, p, trials: int = 200, seed: int = 0) -> str:
        return VERDICTS[self.L.ora_verify(p, trials, seed)]

    def select(self, kind: str, size: int):
        r = self.L.ora_select(KINDS[kind], size)
        return None if r < 0 else IMPLS[r]

    def fill(self, nbytes: int, rank: int, seed: int = 0) -> np.ndarray:
        a = np.empty(nbytes, dtype=np.uint8)
        self.L.ora_fill_pattern(a.ctypes.data, nbytes, rank, seed)
        return a

    def execute(self, p, ins, outs):
        return self.L.ora_execute(p, _ptrs(ins), _ptrs(outs))

    def check(self, kind, s, n, in_place, orig, res) -> int:
        return self.L.ora_check(KINDS[kind], s, n, int(in_place), _ptrs(orig), _ptrs(res))

    def reference_result(self, kind, s, n, ins, outs, nthreads=1):
        self.L.ora_reference_result(KINDS[kind], s, n, _ptrs(ins), _ptrs(outs), nthreads)

    def reduce_scatter(self, dtype: int, op: int, count: int, ins):
        """ora_reduce_scatter over byte buffers ins[i] (n*count elements each)."""
        n = len(ins)
        es = 4 if dtype == 0 else 2
        outs = [np.zeros(count * es, dtype=np.uint8) for _ in range(n)]
        self.L.ora_reduce_scatter(dtype, op, count, n, _ptrs(ins), _ptrs(outs))
        return outs

    def run(self, kind: str, impl: str, s: int, n: int, seed: int = 0):
        """Compile + byte-execute on pattern inputs; returns (inputs, results)."""
        p = self.compile(kind, impl, s, n)
        try:
            in_place = bool(p.contents.in_place)
            in_bytes = s if kind == "allgather" else n * s
            ins = [self.fill(in_bytes, r, seed) for r in range(n)]
            orig = [a.copy() for a in ins]
            outs = [np.full(n * s, 0xA5, dtype=np.uint8) for _ in range(n)]
            self.execute(p, ins, outs)
            return orig, (ins if in_place else outs)
        finally:
            self.free(p)


class Reference:
    """The reference's own compile()/verify_collective()/... (oracle/_ref)."""

    def __init__(self, path: str = REF_LIB):
        if not os.path.exists(path):
            build_oracle()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        L.ref_compile_dump.argtypes = [C.c_char_p, C.c_char_p, C.c_int64, C.c_int, C.c_char_p, C.c_size_t]
        L.ref_metrics.argtypes = [C.c_char_p, C.c_char_p, C.c_int64, C.c_int, C.POINTER(C.c_int * 5)]
        L.ref_traffic.argtypes = [C.c_char_p, C.c_char_p, C.c_int64, C.c_int] + [C.POINTER(C.c_int64)] * 3
        L.ref_validate.argtypes = [C.c_char_p, C.c_char_p, C.c_int64, C.c_int]
        L.ref_verify.argtypes = [C.c_char_p, C.c_char_p, C.c_int64, C.c_int, C.c_uint64]
        L.ref_select.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, C.c_size_t]
        L.ref_execute.argtypes = [C.c_char_p, C.c_char_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]

    def dump(self, kind, impl, s, n):
        cap = 1 << 22
        buf = C.create_string_buffer(cap)
        k = self.L.ref_compile_dump(kind.encode(), impl.encode(), s, n, buf, cap)
        if k == -1:
            raise ValueError("reference compile rejected")
        return buf.raw[:k].decode()

    def metrics(self, kind, impl, s, n):
        out = (C.c_int * 5)()
        assert self.L.ref_metrics(kind.encode(), impl.encode(), s, n, C.byref(out)) == 0
        return list(out)

    def traffic(self, kind, impl, s, n):
        t = (C.c_int64 * 3)()
        gr, gw = (C.c_int64 * n)(), (C.c_int64 * n)()
        assert self.L.ref_traffic(kind.encode(), impl.encode(), s, n, t, gr, gw) == 0
        return list(t), list(gr), list(gw)

    def validate(self, kind, impl, s, n):
        return self.L.ref_validate(kind.encode(), impl.encode(), s, n)

    def verify(self, kind, impl, s, n, seed=0):
        return VERDICTS[self.L.ref_verify(kind.encode(), impl.encode(), s, n, seed)]

    def select(self, kind, size):
        buf = C.create_string_buffer(64)
        rc = self.L.ref_select(kind.encode(), size, buf, 64)
        return None if rc != 0 else buf.value.decode()

    def execute(self, kind, impl, s, n, seed=0):
        in_place = impl.endswith("swap")
        in_bytes = s if kind == "allgather" else n * s
        ins = [splitmix_pattern(in_bytes, r, seed) for r in range(n)]
        outs = [np.full(n * s, 0xA5, dtype=np.uint8) for _ in range(n)]
        rc = self.L.ref_execute(kind.encode(), impl.encode(), s, n, _ptrs(ins), _ptrs(outs))
        if rc != 0:
            raise ValueError("reference compile rejected")
        return ins if in_place else outs
