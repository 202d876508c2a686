"""C-ABI library checks that need no GPU: the in-tree libbolt.so loads, exports
every symbol include/bolt.h declares, and rejects bad arguments on the host
before touching a device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bolt.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bolt_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_1706_10283_b200 import _lib, build
    build.build()
    return _lib.load()


def test_header_symbols_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 20
    from paper_1706_10283_b200 import _lib
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in bolt.h but not exported"
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature in the binding"
    # nothing exported that the header does not declare
    out = os.popen(f"nm -D --defined-only {_lib.LIB_PATH}").read()
    exported = set(re.findall(r"\bT (bolt_\w+)", out))
    assert exported == set(syms), exported ^ set(syms)


def test_version_and_words(lib):
    assert b"sm_100a" in lib.bolt_version()
    assert lib.bolt_codes_words(0, 16) == 0
    assert lib.bolt_codes_words(1, 16) == 16
    assert lib.bolt_codes_words(8, 16) == 16
    assert lib.bolt_codes_words(9, 3) == 6
    assert lib.bolt_codes_words(10, 0) == -1
    assert lib.bolt_codes_words(10, 65) == -1


def test_host_validation(lib):
    from paper_1706_10283_b200._lib import STATUS
    E_SHAPE, E_RANGE, E_NULL = 2, 3, 1
    # shape errors are reported before any device access
    assert lib.bolt_encode(None, 10, 32, 32, None, 0, None, None) == E_SHAPE
    assert "outside 1..64" in lib.bolt_last_error().decode()
    assert lib.bolt_encode(None, 10, 30, 30, None, 8, None, None) == E_SHAPE
    assert "not divisible" in lib.bolt_last_error().decode()
    assert lib.bolt_encode(None, 10, 32, 16, None, 8, None, None) == E_SHAPE
    assert lib.bolt_encode(None, 10, 32, 32, None, 8, None, None) == E_NULL
    assert lib.bolt_encode(None, 0, 32, 32, None, 8, None, None) == 0  # empty is a no-op
    assert lib.bolt_encode_ex(None, 10, 32, 32, None, 8, None, 7, None) == 3  # BOLT_E_RANGE: unknown variant
    assert lib.bolt_quantize_luts(None, 4, 8, ctypes.c_float(0.0), None, None, None) == E_RANGE
    assert lib.bolt_scan(None, 10, 8, None, 4, None, 2, None) == E_NULL
    assert lib.bolt_topk_ex(None, 10, 8, None, 4, 0, 0, 0, None, None, 0, 0, None) == E_NULL
    k = ctypes.c_void_p(16)
    assert lib.bolt_topk_ex(k, 10, 8, k, 4, 0, 0, 0, None, None, 0, 0, None) == E_SHAPE
    assert lib.bolt_topk_ex(k, 10, 8, k, 4, 129, 0, 0, None, None, 0, 0, None) == E_SHAPE
    assert lib.bolt_topk_ex(k, 10, 8, k, 4, 10, 2, 0, None, None, 0, 0, None) == E_RANGE
    assert lib.bolt_topk_ex(k, 10, 8, k, 4, 10, 0, 0, None, None, 0, 7, None) == E_RANGE
    assert lib.bolt_topk_ex(k, 10, 8, k, 4, 10, 0, 1 << 48, None, None, 0, 0, None) == E_RANGE
    assert lib.bolt_topk_merge(None, 20000, 4, 100, None, None) == E_SHAPE
    assert lib.bolt_topk_merge(None, 2, 4, 129, None, None) == E_SHAPE
    assert set(STATUS) == set(range(8))


def test_workspace_sizing_host(lib):
    # the plan is a pure function of the shapes (and SM count): partial lists
    # [parts][nq][k] u64, then the shared per-query threshold words: one
    # (PRMT), 33 (small-batch PRMT kernel, nq < 64 and m in {8,16,32}: k-th
    # value + 32 minima slots), 9 nq + 4 + rparts ceil(nq / 128) (tcgen05: k-th
    # value words, 16 B aligned rows of 8 union-group words, finished-partition
    # counters; for k > 32 the 9 nq + 4 words become 4 nq group words)
    for n, m, nq, k, variant in [(10, 8, 4, 10, 1), (1_000_000, 16, 10_000, 10, 1), (10**8, 16, 1, 100, 1),
                                 (5000, 12, 8, 10, 1), (1_000_000, 16, 10_000, 10, 2), (777, 32, 300, 32, 2)]:
        ws = lib.bolt_topk_workspace_bytes_ex(n, m, nq, k, variant)
        rv, parts = ctypes.c_int(0), ctypes.c_int(0)
        assert lib.bolt_topk_plan(n, m, nq, k, variant, ctypes.byref(rv), ctypes.byref(parts)) == 0
        assert rv.value == variant
        p = parts.value
        if variant == 2:
            expect = p * nq * k * 8 + (9 * nq + 4 + (p // 2) * -(-nq // 128)) * 4
        elif nq < 64 and m in (8, 16, 32):
            expect = p * nq * k * 8 + 33 * nq * 4
        else:
            expect = 0 if p == 1 else p * nq * k * 8 + nq * 4
        assert ws == expect, (n, m, nq, k, variant, p, ws)
        assert 1 <= p <= 16384


def test_c_example_builds(lib, tmp_path):
    """examples/search.c uses the C ABI alone (no Python): it compiles and
    links against bolt.h and libbolt.so (run on a GPU by hand or by tools)."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    out = tmp_path / "search"
    inc = os.path.join(ROOT, "include")
    libdir = os.path.join(ROOT, "paper_1706_10283_b200")
    r = subprocess.run(["gcc", "-O2", "-std=c11", "-Wall", "-Werror", f"-I{inc}", "-I/usr/local/cuda/include",
                        "-o", str(out), os.path.join(ROOT, "examples", "search.c"), f"-L{libdir}", "-lbolt",
                        f"-Wl,-rpath,{libdir}", "-L/usr/local/cuda/lib64", "-lcudart"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
