"""C++ host code over the C ABI (include/kvmix_b200.hpp): the reference's hot-path API
written the way the reference's callers write it, compiled with g++ and run against the
reference library itself (tests/cpp/shim_parity.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _compile(out):
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"),
           os.path.join(ROOT, "tests", "cpp", "shim_parity.cpp"), "-o", out,
           "-L", os.path.join(ROOT, "paper_2506_08018_b200"), "-lkvmix_b200",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2506_08018_b200"),
           "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-Wl,-rpath," + os.path.join(CUDA, "lib64"), "-ldl"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_shim_compiles(tmp_path):
    """The header-only shim and the parity program build against libkvmix_b200 (CPU tier)."""
    _compile(str(tmp_path / "shim_parity"))


@pytest.mark.gpu
def test_shim_parity_against_reference(cuda, tmp_path):
    ref = os.path.join(ROOT, "oracle", "_ref", "libkvmix_ref.so")
    if not os.path.exists(ref):
        pytest.fail("oracle/_ref/libkvmix_ref.so missing: run __graft_entry__.build() where /root/reference exists")
    exe = str(tmp_path / "shim_parity")
    _compile(exe)
    r = subprocess.run([exe, ref], capture_output=True, text=True, cwd=ROOT, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
