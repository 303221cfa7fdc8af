"""cecoll_program_parse reads program text from outside (the reference's
dump_program output, or hand-written programs): random mutations of the
golden dumps must parse or be rejected with InvalidArgument — never crash —
and whatever parses must go through validate / metrics / dump (CPU only)."""
import json
import os
import random

import paper_2511_06605_b200 as cc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _dumps():
    with open(os.path.join(ROOT, "tests", "golden", "programs.json")) as f:
        return [e for e in json.load(f)["programs"] if "dump" in e and e["n"] <= 8]


def _mutate(rng, text):
    lines = text.splitlines()
    op = rng.randrange(7)
    i = rng.randrange(len(lines))
    if op == 0:  # drop a line
        del lines[i]
    elif op == 1:  # duplicate a line
        lines.insert(i, lines[i])
    elif op == 2:  # swap two lines
        j = rng.randrange(len(lines))
        lines[i], lines[j] = lines[j], lines[i]
    elif op == 3:  # corrupt one field
        f = lines[i].split("\t")
        k = rng.randrange(len(f))
        f[k] = rng.choice(["", "-", "x", "-1", "999999999999999999999", "g9.in[0+1]", "g0.out[-5+3]",
                           "q0(g0e0)", "copy", "swap", "poll", "signal", "broadcast", "1e9", "\x00"])
        lines[i] = "\t".join(f)
    elif op == 4:  # truncate a line
        lines[i] = lines[i][: rng.randrange(len(lines[i]) + 1)]
    elif op == 5:  # random bytes
        lines[i] = "".join(chr(rng.randrange(32, 127)) for _ in range(rng.randrange(40)))
    else:  # change a number somewhere
        f = lines[i].split("\t")
        k = rng.randrange(len(f))
        f[k] = "".join(ch if not ch.isdigit() else str(rng.randrange(10)) for ch in f[k])
        lines[i] = "\t".join(f)
    return "\n".join(lines) + ("\n" if rng.random() < 0.9 else "")


def test_parse_survives_mutated_reference_text():
    rng = random.Random(2511)
    dumps = _dumps()
    parsed = rejected = 0
    for _ in range(3000):
        e = rng.choice(dumps)
        text = e["dump"]
        for _ in range(rng.randrange(1, 4)):
            text = _mutate(rng, text)
        try:
            p = cc.Program.parse(text, e["kind"], e["s"], e["n"])
        except cc.InvalidArgument:
            rejected += 1
            continue
        parsed += 1
        p.validate()  # None or the first violation; must not crash
        p.metrics()
        p.traffic()
        p.dump()
    assert parsed > 100 and rejected > 100, (parsed, rejected)


def test_parse_rejects_bad_parameters():
    e = _dumps()[0]
    for n in (0, -3, 5000):
        try:
            cc.Program.parse(e["dump"], e["kind"], e["s"], n)
            raise AssertionError(f"accepted gpu_count {n}")
        except cc.InvalidArgument:
            pass


def test_program_api_survives_random_arguments():
    """compile / select / metrics / traffic / validate / dump through the C
    ABI with hostile arguments: errors, never crashes or runaway work."""
    import ctypes as C

    L = cc.lib()
    rng = random.Random(606)
    ok = 0
    for _ in range(3000):
        kind = rng.choice([0, 1, 2, -1, 7])
        impl = rng.choice(list(range(-3, 13)))
        s = rng.choice([0, -1, 1, 15, 4096, 1 << 40, -(1 << 62)])
        n = rng.choice([0, 1, 2, 3, 8, 16, 33, 1025, -5])
        lanes = rng.choice([0, 1, 2, 16, 64, -1])
        h = C.c_void_p()
        st = L.cecoll_program_compile(kind, impl, s, n, lanes, C.byref(h))
        L.cecoll_select(kind, s, n, rng.choice([0, 1, 8]))
        L.cecoll_reference_select(kind, s)
        if st != 0:
            assert not h.value
            continue
        ok += 1
        p = cc.Program({0: "allgather", 1: "alltoall"}[kind], None, s, n, _handle=h)
        p.metrics()
        p.traffic()
        p.validate(max(1, lanes))
        if n <= 16:
            p.dump()
    assert ok > 50, ok


def test_runtime_entry_points_reject_null_handles():
    """Every runtime entry point checks its handles before touching them
    (no CUDA needed: the checks come first): null communicators inside the
    arrays, null plans, null outputs -> CECOLL_INVALID_ARGUMENT, no crash."""
    import ctypes as C

    L = cc.lib()
    vp = C.c_void_p
    null_comms = (vp * 2)(None, None)
    bufs = (vp * 2)(None, None)
    out = vp()
    L.cecoll_plan_create.argtypes = [C.POINTER(vp), C.c_int, C.c_int, C.POINTER(vp), C.POINTER(vp), C.c_size_t,
                                     C.c_int, C.POINTER(vp)]
    assert L.cecoll_plan_create(null_comms, 2, 0, bufs, bufs, 4096, 0, C.byref(out)) == 1
    assert L.cecoll_plan_create(null_comms, 2, 7, bufs, bufs, 4096, 0, C.byref(out)) == 1  # unknown kind
    assert L.cecoll_plan_create_program(null_comms, 2, vp(1), bufs, bufs, C.byref(out)) == 1
    assert L.cecoll_plan_launch(None, None) == 1
    assert L.cecoll_plan_arm(None) == 1
    assert L.cecoll_plan_trigger(None, None) == 1
    assert L.cecoll_plan_disarm(None) == 1
    assert L.cecoll_plan_destroy(None) == 1
    assert L.cecoll_comm_destroy(None) == 1
    code = C.c_int(0)
    assert L.cecoll_comm_get_async_error(None, C.byref(code)) == 1
    assert L.cecoll_mem_alloc(None, 4096, C.byref(out)) == 1
    assert L.cecoll_mem_free(None, None) == 1
    assert L.cecoll_register(None, None, 0) == 1
    assert L.cecoll_deregister(None, None) == 1
    assert L.cecoll_collective_n(0, null_comms, 2, bufs, bufs, 4096, 0, None) == 1
    assert L.cecoll_reduce_scatter_n(null_comms, 2, bufs, bufs, 1024, 1, 0, 0, None) == 1
    assert L.cecoll_allgather(None, None, 4096, 0, None, None) == 1
    assert b"null" in L.cecoll_last_error()
