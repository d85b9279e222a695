"""C++ test of the reference-side binding logic (include/rtn_adapter.hpp, used by
INTEGRATION.md's MlpBatchedEval replacement) through the C-ABI:
tests/cpp/test_adapter.cpp. Built here with the system g++ against the in-tree
librtn_mpc.so and the oracle (test infrastructure)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_adapter.cpp")
LIBDIR = os.path.join(ROOT, "paper_2203_07747_b200")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    from paper_2203_07747_b200 import build
    build.build_library()
    out = str(tmp_path_factory.mktemp("cpp") / "test_adapter")
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cmd = [cxx, "-std=c++17", "-O2", "-pthread", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "oracle"),
           SRC, os.path.join(ROOT, "oracle", "resmpc_oracle.cpp"), "-L", LIBDIR, "-lrtn_mpc",
           f"-Wl,-rpath,{LIBDIR}", "-o", out]
    subprocess.run(cmd, check=True)
    return out


def test_adapter_builds_and_fails_loudly_without_a_device(binary):
    from conftest import _has_gpu
    if _has_gpu():
        pytest.skip("a device is present: the full scenario runs in test_adapter_scenarios_on_device")
    r = subprocess.run([binary, "--no-device"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_adapter_scenarios_on_device(binary):
    r = subprocess.run([binary], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
