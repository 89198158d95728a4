"""CPU tests of the drop-in boundary: header conformance with the reference, the C-ABI
symbol table, and the no-fallback contract (no GPU here -> every entry refuses)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
GXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def _compile(include_dir):
    src = os.path.join(ROOT, "tests", "cpp", "api_conformance.cpp")
    return subprocess.run([GXX, "-std=c++20", "-fsyntax-only", "-I", include_dir, src], capture_output=True, text=True)


def test_conformance_tu_compiles_against_our_headers():
    r = _compile(os.path.join(ROOT, "include"))
    assert r.returncode == 0, r.stderr


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference tree not present (GPU box)")
def test_conformance_tu_compiles_against_reference_headers():
    r = _compile(REF_INC)
    assert r.returncode == 0, r.stderr


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "hps_gpu.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(hps_(?:gpu_|plan_|shard_|estimate_|key_hash_host|fastmod)\w*)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    from paper_2210_08803_b200 import _lib
    lib = _lib.load()
    syms = _declared_symbols()
    assert len(syms) >= 45
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) <= set(_lib.SIGNATURES), sorted(set(syms) - set(_lib.SIGNATURES))


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2210_08803_b200 import _lib
    lib = _lib.load()
    h = C.c_void_p()
    st = lib.hps_gpu_ctx_create(0, None, C.byref(h))
    assert st == _lib.E_NO_DEVICE
    assert b"no CPU fallback" in lib.hps_gpu_last_error_message()
    assert lib.hps_gpu_status_string(st) == b"NoDevice"
    assert lib.hps_gpu_abi_version() == 1


def test_sm100a_only_binary():
    so = os.path.join(ROOT, "paper_2210_08803_b200", "libhps_gpu.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs
