"""The C ABI driven from C++ alone across processes (tools/mp_selftest.cpp):
forked processes exchange blobs through shared memory, register a
library-owned window and run every implementation, byte-checked, then run
cecoll_tune and check that every process installed the same table."""
import os
import shutil
import subprocess

import pytest

import paper_2511_06605_b200 as cc

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tools", "mp_selftest")


def _build():
    src = os.path.join(ROOT, "tools", "mp_selftest.cpp")
    if os.path.exists(EXE) and os.path.getmtime(EXE) >= os.path.getmtime(src):
        return
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    libdir = os.path.dirname(cc.LIB_PATH)
    subprocess.run([nvcc, "-O2", "-std=c++17", src, f"-I{os.path.join(ROOT, 'include')}", f"-L{libdir}", "-lcecoll",
                    "-Xlinker", f"-rpath,{libdir}", "-o", EXE], check=True)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("nprocs,chunk", [(2, 65536 + 48), (4, 4099)])
def test_cpp_processes_every_implementation(nprocs, chunk):
    _build()
    r = subprocess.run([EXE, str(nprocs), str(chunk)], capture_output=True, text=True, timeout=500)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all implementations bit-exact" in r.stdout
    assert r.stdout.count("PASS") >= 15 and "FAIL" not in r.stdout
    assert "tune      same table      PASS" in r.stdout  # cecoll_tune from C, agreed across processes
