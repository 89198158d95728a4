"""Runs the C++ host-API test binary (tests/cpp/test_gpu_api.cpp, hps::gpu wrappers)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_host_api():
    exe = os.path.join(ROOT, "tests", "cpp", "test_gpu_api")
    assert os.path.exists(exe), "build() compiles tests/cpp/test_gpu_api"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "passed" in r.stdout


def test_cpp_sharded_c_abi():
    """tests/cpp/test_dist_api.cpp: a C++ caller drives hps_gpu_dist_* over NCCL (world of
    one) and the loopback transport (world of two, a thread per rank)."""
    exe = os.path.join(ROOT, "tests", "cpp", "test_dist_api")
    assert os.path.exists(exe), "build() compiles tests/cpp/test_dist_api"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "passed" in r.stdout
