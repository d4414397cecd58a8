"""CPU-side checks of the product library (no GPU needed): it builds for
sm_100a, loads, exports every symbol include/rairs.h declares, carries sm_100a
SASS with no legacy tensor path, and the binding rejects bad arguments before
touching the device."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rb():
    from paper_2601_07183_b200 import _lib
    _lib.build_library()
    import paper_2601_07183_b200
    return paper_2601_07183_b200


def header_symbols():
    src = open(os.path.join(ROOT, "include", "rairs.h")).read()
    return sorted(set(re.findall(r"\b(rairs_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_match_binding_list(rb):
    assert header_symbols() == sorted(rb.EXPORTED_SYMBOLS)


def test_library_exports_every_header_symbol(rb):
    out = subprocess.check_output(["nm", "-D", "--defined-only", rb.LIB_PATH]).decode()
    exported = set(line.split()[-1] for line in out.splitlines() if " T " in line)
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, f"missing exports: {missing}"
    lib = rb.lib()
    for s in header_symbols():
        assert hasattr(lib, s)


def test_library_is_sm100a(rb):
    out = subprocess.check_output(["cuobjdump", "--list-elf", rb.LIB_PATH]).decode()
    assert "sm_100a" in out
    sass = subprocess.check_output(["cuobjdump", "-sass", rb.LIB_PATH]).decode()
    assert not re.search(r"(?<![A-Z])HMMA", sass)   # no legacy mma.sync path
    assert "UTCHMMA" in sass                       # tcgen05.mma (coarse TF32 GEMM)
    assert "UTCIMMA" in sass                       # tcgen05.mma kind::i8 (list-major scan)
    assert "STTM" in sass                          # tcgen05.st (one-hot A operand in TMEM)
    assert "UTMALDG" in sass                       # TMA tensor loads
    assert "LDTM" in sass                          # tcgen05.ld from TMEM


def test_version_and_error_channel(rb):
    lib = rb.lib()
    assert b"sm_100a" in lib.rairs_version()
    # NULL index -> RAIRS_E_INVALID before any device work
    st = lib.rairs_search(None, None, 1, 10, 1, 1, None, None, None, None)
    assert st == -1
    assert b"index" in lib.rairs_last_error()


def test_default_params(rb):
    from paper_2601_07183_b200.index import make_params
    p = make_params(1024, 64)
    assert (p.nlist, p.M, p.nbits, p.assignment, p.n_cands, p.strict) == (1024, 64, 4, 1, 10, 0)
    assert abs(p.lambda_ - 0.5) < 1e-9
