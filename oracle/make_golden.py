"""Generate tests/golden/ fixtures from the reference itself.

Run here (the reference tree must be present):  python oracle/make_golden.py

Everything recorded comes from oracle/_ref/libdmasim_ref.so, i.e. the
reference's own unmodified compile()/dump_program()/static_metrics()/
account_traffic()/validate_program()/verify_collective()/
select_implementation() (proj/src/{compiler,program,verifier}.cpp), plus the
byte executor of oracle/ref_shim.cpp run over the reference's compiled
CommandProgram. The fixtures travel to the GPU box; /root/reference does not.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import IMPLS_FOR, Reference  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def sha(data: bytes) -> str:
    return hashlib.sha256(data).hexdigest()


def main() -> None:
    ref = Reference()
    os.makedirs(OUT, exist_ok=True)

    # 1. Command programs: full dump text at n in {2,3,4,8}, digests up to 16.
    programs = []
    for kind in ("allgather", "alltoall"):
        for impl in IMPLS_FOR[kind]:
            for n in range(2, 17):
                for s in (1024, 4096, 1 << 20):
                    text = ref.dump(kind, impl, s, n)
                    traffic, gr, gw = ref.traffic(kind, impl, s, n)
                    entry = {
                        "kind": kind,
                        "impl": impl,
                        "n": n,
                        "s": s,
                        "dump_sha256": sha(text.encode()),
                        "dump_lines": text.count("\n"),
                        "metrics": ref.metrics(kind, impl, s, n),
                        "traffic": traffic,
                        "per_gpu_read": gr,
                        "per_gpu_write": gw,
                        "valid": ref.validate(kind, impl, s, n) == 0,
                    }
                    if s == 4096 and n in (2, 3, 4, 8):
                        entry["dump"] = text
                    if s == 1024 and n in (2, 3, 4, 5, 8):
                        entry["verdict"] = ref.verify(kind, impl, s, n, seed=0)
                    programs.append(entry)
    # Rejections (compiler.cpp:142-145, 173-179, 212-213, 289-291; program.cpp:31-38).
    rejects = []
    for kind, impl, s, n in [
        ("alltoall", "bcst", 4096, 8),
        ("allgather", "swap", 4096, 8),
        ("allgather", "pcpy", 4096, 20),
        ("allgather", "pcpy", 0, 8),
        ("alltoall", "b2b", 4096, 1),
        ("allgather", "prelaunch_swap", 4096, 8),
    ]:
        try:
            ref.dump(kind, impl, s, n)
            ok = True
        except ValueError:
            ok = False
        rejects.append({"kind": kind, "impl": impl, "s": s, "n": n, "accepted": ok})
    with open(os.path.join(OUT, "programs.json"), "w") as f:
        json.dump({"programs": programs, "rejects": rejects}, f, indent=0, sort_keys=True)

    # 2. select_implementation step function (compiler.cpp:305-318).
    sizes = [512, 1023, 1 << 10]
    for b in (64 << 10, 256 << 10, 1 << 20, 4 << 20, 512 << 20, 1 << 30):
        sizes += [b - 1, b, b + 1]
    sizes += [8 << 30]
    select = {kind: [[sz, ref.select(kind, sz)] for sz in sizes] for kind in ("allgather", "alltoall")}
    with open(os.path.join(OUT, "select.json"), "w") as f:
        json.dump(select, f, indent=1, sort_keys=True)

    # 3. Byte digests of the reference program run on splitmix inputs.
    digests = []
    for kind in ("allgather", "alltoall"):
        for impl in IMPLS_FOR[kind]:
            for n in (2, 3, 4, 5, 8):
                for s in (1024, 1000, 4099, 65536):
                    for seed in (0, 1):
                        if seed == 1 and s != 1024:
                            continue
                        res = ref.execute(kind, impl, s, n, seed)
                        digests.append({
                            "kind": kind, "impl": impl, "n": n, "s": s, "seed": seed,
                            "sha256": [sha(r.tobytes()) for r in res],
                        })
    with open(os.path.join(OUT, "digests.json"), "w") as f:
        json.dump(digests, f, indent=0, sort_keys=True)
    print(f"wrote {len(programs)} programs, {len(digests)} digests to {OUT}")
    baseline_configs(ref)


# BASELINE.json configs at their exact sizes (SURVEY.md §8 sizing): C0 all-gather
# n=8 s=1 MiB, C1 all-to-all n=8 s=8 MiB (the bench headline), C4 all-gather
# n=8 s=256 MiB. Every reference implementation of the collective is executed
# (the reference's compile() + byte executor) on the seeded splitmix inputs and
# the sha256 of every rank's output is recorded (seeds 0 and 1).
BASELINE_CASES = [
    ("C0", "allgather", 8, 1 << 20, (0, 1)),
    ("C1", "alltoall", 8, 8 << 20, (0,)),
    ("C4", "allgather", 8, 256 << 20, (0,)),
]


def baseline_configs(ref=None) -> None:
    import gc

    ref = ref or Reference()
    cases = []
    for name, kind, n, s, seeds in BASELINE_CASES:
        for impl in IMPLS_FOR[kind]:
            for seed in seeds:
                res = ref.execute(kind, impl, s, n, seed)
                cases.append({"config": name, "kind": kind, "impl": impl, "n": n, "s": s, "seed": seed,
                              "sha256": [sha(memoryview(r)) for r in res]})
                del res
                gc.collect()
                print(name, impl, seed, cases[-1]["sha256"][0][:16], flush=True)
    with open(os.path.join(OUT, "baseline_configs.json"), "w") as f:
        json.dump(cases, f, indent=0, sort_keys=True)
    print(f"wrote {len(cases)} baseline-config digests to {OUT}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "baseline":
        baseline_configs()
    else:
        main()
