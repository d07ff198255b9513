"""C-ABI boundary checks that need no GPU: libuzip.so loads, exports every
symbol include/uzip.h declares, sizes agree with the oracle's closed forms,
host-side argument validation returns the documented errors, and the product
path is independent of oracle/ (no import, no shared symbol)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def uz():
    import paper_2604_17172_b200 as uz
    uz.build()
    return uz


def _declared():
    hdr = open(os.path.join(ROOT, "include", "uzip.h")).read()
    return sorted(set(re.findall(r"UZIP_API[^;(]*?\b(uzip_\w+)\s*\(", hdr, flags=re.S)))


def test_exports_every_declared_symbol(uz):
    names = _declared()
    assert len(names) >= 17
    out = subprocess.check_output(["nm", "-D", "--defined-only", uz.LIB_PATH], text=True)
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(names) <= exported, set(names) - exported
    for n in names:
        assert hasattr(uz.lib(), n)
    assert set(uz.EXPORTED) == set(names)


def test_version_and_status_strings(uz):
    assert "sm_100a" in uz.version()
    for code in range(10):
        assert uz.status_string(code)


@pytest.mark.parametrize("dtype", [0, 1, 2])
@pytest.mark.parametrize("n", [0, 1, 4095, 4096, 4097, 2097152, 536870912])
def test_compress_bound_matches_oracle(uz, orc, dtype, n):
    assert uz.compress_bound(n, dtype) == orc.compress_bound(n, dtype)
    for B in (1024, 2048):
        assert uz.compress_bound(n, dtype, block_symbols=B) == orc.compress_bound(n, dtype, block_symbols=B)
    assert uz.compress_bound(n, dtype, global_table=True) == orc.compress_bound(n, dtype, global_table=True)
    assert uz.workspace_bytes(n, dtype) >= 64


def test_host_validation_errors(uz):
    l = uz.lib()
    p = uz.CodecParams(4096, 0, 0, 0)
    vp = ctypes.c_void_p
    # unsupported dtype
    assert l.uzip_compress(vp(16), 10, 7, vp(16), 1 << 20, None, vp(16), 1 << 20, ctypes.byref(p), None) == \
        uz.ERR_UNSUPPORTED_DTYPE
    # null / misaligned pointers
    assert l.uzip_compress(None, 10, 0, vp(16), 1 << 20, None, vp(16), 1 << 20, ctypes.byref(p), None) == \
        uz.ERR_INVALID_ARG
    assert l.uzip_compress(vp(17), 10, 0, vp(16), 1 << 20, None, vp(16), 1 << 20, ctypes.byref(p), None) == \
        uz.ERR_INVALID_ARG
    # capacity
    assert l.uzip_compress(vp(16), 4096 * 4, 0, vp(16), 100, None, vp(16), 1 << 20, ctypes.byref(p), None) == \
        uz.ERR_CAPACITY
    # unsupported block size on the GPU path
    bad = uz.CodecParams(64, 0, 0, 0)
    assert l.uzip_compress(vp(16), 10, 0, vp(16), 1 << 20, None, vp(16), 1 << 20, ctypes.byref(bad), None) == \
        uz.ERR_INVALID_ARG
    assert uz.compress_bound(10, 0, block_symbols=64) == 0
    # decompress: null status word
    assert l.uzip_decompress(vp(16), 100, vp(16), 10, 0, None, vp(16), 64, None) == uz.ERR_INVALID_ARG
    assert l.uzip_decompress(vp(16), 100, vp(16), 10, 9, vp(16), vp(16), 64, None) == uz.ERR_UNSUPPORTED_DTYPE


def test_product_independent_of_oracle(uz):
    pkg = os.path.join(ROOT, "paper_2604_17172_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cc")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src and "uzip_oracle" not in src, f
    out = subprocess.check_output(["nm", "-D", uz.LIB_PATH], text=True)
    assert "uzo_" not in out
