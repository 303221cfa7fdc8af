"""The product's planner (libcecoll.so, C ABI) against the reference's goldens.

CPU only: the planner emits the exact command program the executors lower
onto the GPU, so its dump_program text, metrics and traffic must equal the
reference's (tests/golden/programs.json, from proj/src/compiler.cpp).
"""
import json
import os
import re

import pytest

import paper_2511_06605_b200 as cc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def test_library_exports_every_declared_symbol():
    L = cc.lib()
    with open(os.path.join(ROOT, "include", "cecoll.h")) as f:
        header = f.read()
    declared = set(re.findall(r"\b(cecoll_[a-z_0-9]+)\s*\(", header))
    declared -= {"cecoll_exchange_fn"}
    assert declared, "no declarations parsed"
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert set(cc.EXPORTED_SYMBOLS) <= declared


def test_programs_match_reference_goldens():
    with open(os.path.join(GOLDEN, "programs.json")) as f:
        data = json.load(f)
    import hashlib

    for e in data["programs"]:
        p = cc.Program(e["kind"], e["impl"], e["s"], e["n"])
        text = p.dump()
        assert hashlib.sha256(text.encode()).hexdigest() == e["dump_sha256"], (e["kind"], e["impl"], e["n"])
        if "dump" in e:
            assert text == e["dump"]
        m = p.metrics()
        assert [m[k] for k in ("data_commands", "sync_commands", "poll_commands", "engines_used", "doorbells")] == e[
            "metrics"
        ]
        t = p.traffic()
        assert [t["read"], t["write"], t["link"]] == e["traffic"]
        assert t["rank_read"] == e["per_gpu_read"] and t["rank_write"] == e["per_gpu_write"]
        assert p.validate() is None
        assert e["valid"]


def test_rejections_match_reference():
    with open(os.path.join(GOLDEN, "programs.json")) as f:
        data = json.load(f)
    for r in data["rejects"]:
        if r["accepted"]:
            cc.Program(r["kind"], r["impl"], r["s"], r["n"])
        else:
            with pytest.raises(cc.InvalidArgument):
                cc.Program(r["kind"], r["impl"], r["s"], r["n"])


def test_reference_select_table():
    with open(os.path.join(GOLDEN, "select.json")) as f:
        table = json.load(f)
    for kind, rows in table.items():
        for size, name in rows:
            assert cc.reference_select(kind, size) == name, (kind, size)


def test_impl_names_round_trip():
    L = cc.lib()
    for name, v in cc.IMPLS.items():
        if name == "auto":
            continue
        assert L.cecoll_parse_impl(name.encode()) == v
        if name != "baseline":
            assert cc.impl_name(v) == name
    assert L.cecoll_parse_impl(b"nope") == -2
    assert L.cecoll_impl_valid_for(1, 0) == 1 and L.cecoll_impl_valid_for(1, 1) == 0  # bcst: AG only
    assert L.cecoll_impl_valid_for(2, 1) == 1 and L.cecoll_impl_valid_for(2, 0) == 0  # swap: AA only


def test_prelaunch_adds_one_poll_per_lane_and_keeps_traffic():
    base = cc.Program("allgather", "pcpy", 4096, 8)
    pre = cc.Program("allgather", "prelaunch_pcpy", 4096, 8)
    mb, mp = base.metrics(), pre.metrics()
    assert mp["poll_commands"] == mb["engines_used"] == 56
    assert mp["data_commands"] == mb["data_commands"]
    assert pre.traffic() == base.traffic()
    assert all(line.split("\t")[2] == "poll" for line in pre.dump().splitlines() if line.split("\t")[1] == "0")


def test_engine_budget_is_enforced():
    with pytest.raises(cc.InvalidArgument):
        cc.Program("allgather", "pcpy", 4096, 8, lanes_per_rank=6)  # needs n-1 = 7 lanes
    cc.Program("allgather", "b2b", 4096, 8, lanes_per_rank=1)


def test_comm_init_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(cc.CecollError):
        cc.Comm.init_all([0, 0])


def test_parse_reference_dump_round_trips():
    with open(os.path.join(GOLDEN, "programs.json")) as f:
        data = json.load(f)
    seen = 0
    for e in data["programs"]:
        if "dump" not in e:
            continue
        p = cc.Program.parse(e["dump"], e["kind"], e["s"], e["n"])
        assert p.dump() == e["dump"]
        m = p.metrics()
        assert [m[k] for k in ("data_commands", "sync_commands", "poll_commands", "engines_used", "doorbells")] == e[
            "metrics"
        ]
        assert p.validate() is None
        seen += 1
    assert seen == 48


def test_parse_rejects_malformed_text():
    with pytest.raises(cc.InvalidArgument):
        cc.Program.parse("q0(g0e0)\t0\tfrobnicate\t-\t-\t0\t-\n", "allgather", 1024, 2)
    with pytest.raises(cc.InvalidArgument):
        cc.Program.parse("q0(g0e0)\t0\tcopy\tg0.in[0+1024]\n", "allgather", 1024, 2)
    # Out-of-bounds programs parse but do not validate (program.cpp:85-94).
    bad = cc.Program.parse("q0(g0e0)\t0\tcopy\tg0.in[0+1024]\tg1.out[4096+1024]\t1024\t-\n"
                           "q0(g0e0)\t1\tsignal\t-\t-\t0\t0\n", "allgather", 1024, 2)
    assert "out of declared bounds" in bad.validate()


def _ref_dump(kind, impl, s, n):
    with open(os.path.join(GOLDEN, "programs.json")) as f:
        for e in json.load(f)["programs"]:
            if (e["kind"], e["impl"], e["s"], e["n"]) == (kind, impl, s, n) and "dump" in e:
                return e["dump"]
    raise KeyError((kind, impl, s, n))


def _mutate(text, fn):
    lines = [line.split("\t") for line in text.splitlines()]
    fn(lines)
    return "\n".join("\t".join(f) for f in lines) + "\n"


def test_validate_catches_engine_overflow_and_duplicates():
    # test_program.cpp:94-110: engine index past the budget; two queues on one engine.
    text = _ref_dump("allgather", "pcpy", 4096, 8)
    over = _mutate(text, lambda ls: [f.__setitem__(0, "q0(g0e16)") for f in ls if f[0] == "q0(g0e0)"])
    assert "engine overflow" in cc.Program.parse(over, "allgather", 4096, 8).validate(16)
    dup = _mutate(text, lambda ls: [f.__setitem__(0, "q1(g0e0)") for f in ls if f[0] == "q1(g0e1)"])
    assert "share one engine" in cc.Program.parse(dup, "allgather", 4096, 8).validate(16)


def test_validate_requires_trailing_signal_and_matching_triggers():
    # test_program.cpp:112-138: dropped AtomicSignal; trigger slots vs polls.
    text = _ref_dump("allgather", "pcpy", 4096, 8)
    dropped = _mutate(text, lambda ls: ls.remove(next(f for f in ls if f[0].startswith("q3(") and f[2] == "signal")))
    assert "unsignaled queue" in cc.Program.parse(dropped, "allgather", 4096, 8).validate(16)
    pre = _ref_dump("allgather", "prelaunch_pcpy", 4096, 8)
    assert cc.Program.parse(pre, "allgather", 4096, 8).validate(16) is None
    late_poll = _mutate(pre, lambda ls: ls.insert(2, ["q0(g0e0)", "1", "poll", "-", "-", "0", "100999"]))
    assert "poll must precede" in cc.Program.parse(late_poll, "allgather", 4096, 8).validate(16)


def test_validate_rejects_overlap_and_same_gpu_swap():
    text = _ref_dump("alltoall", "pcpy", 4096, 4)
    overlap = _mutate(text, lambda ls: [f.__setitem__(4, f[3].replace(".in[", ".in[")) for f in ls
                                        if f[0] == "q0(g0e0)" and f[2] == "copy"])
    assert "overlap" in cc.Program.parse(overlap, "alltoall", 4096, 4).validate(16)
    swap = _ref_dump("alltoall", "swap", 4096, 4)
    same = _mutate(swap, lambda ls: [f.__setitem__(4, f[3]) for f in ls if f[2] == "swap"][:1])
    assert "distinct gpus" in cc.Program.parse(same, "alltoall", 4096, 4).validate(16)


def test_b200_selector_is_total_and_valid():
    for kind in ("allgather", "alltoall"):
        for ndev in (1, 2, 8):
            for k in range(10, 33):
                impl = cc.select(kind, 1 << k, 8, ndev)
                assert impl == "sm" or impl in cc.IMPLS_FOR[kind]
    assert cc.select("allgather", 1 << 30, 8, 1) == "sm"
    assert cc.select("alltoall", 4096, 8, 8) == "sm"


def test_header_is_plain_c_and_links(tmp_path):
    """include/cecoll.h is the drop-in boundary for C callers (and cgo / JNI /
    ctypes bindings): a C99 program compiles against it with -pedantic and
    links against libcecoll.so; the program API runs without a GPU."""
    import shutil
    import subprocess

    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no C compiler")
    src = tmp_path / "t.c"
    src.write_text(
        '#include "cecoll.h"\n#include <stdio.h>\n'
        "int main(void) {\n"
        "  cecoll_program_t p = 0; int64_t m[5];\n"
        "  if (cecoll_program_compile(CECOLL_ALLGATHER, CECOLL_IMPL_PCPY, 4096, 8, 16, &p) != CECOLL_SUCCESS) return 1;\n"
        "  if (cecoll_program_metrics(p, m) != CECOLL_SUCCESS) return 2;\n"
        '  printf("%lld %s\\n", (long long)m[0], cecoll_impl_name(CECOLL_IMPL_PULL));\n'
        "  cecoll_program_free(p);\n  return 0;\n}\n")
    libdir = os.path.dirname(cc.LIB_PATH)
    exe = tmp_path / "t"
    subprocess.run([gcc, "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", f"-I{os.path.join(ROOT, 'include')}",
                    str(src), f"-L{libdir}", "-lcecoll", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    assert out == ["56", "pull"]  # n(n-1) copies (test_program.cpp:29-43)
