"""The C-ABI library loads and exports every symbol include/tt_hotpath.h declares; host-side
validation (no GPU needed: every call here fails validation before touching CUDA)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tt_hotpath.h")
DEBUG_HEADER = os.path.join(ROOT, "include", "tt_hotpath_debug.h")
LIB = os.path.join(ROOT, "paper_2509_11890_b200", "libtt_hotpath.so")


def declared_functions():
    src = open(HEADER).read() + open(DEBUG_HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tt_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_hot_path(lib):
    names = declared_functions()
    for n in ["tt_local_matvec", "tt_local_matvec_batched", "tt_interface_left",
              "tt_interface_right", "tt_sweep_interfaces", "tt_operator_apply",
              "tt_local_matvec_workspace_size", "tt_sweep_als", "tt_status_string",
              "tt_last_error_message"]:
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    for n in declared_functions():
        assert hasattr(lib, n), n


def test_python_binding_names_match_header():
    import paper_2509_11890_b200 as tt
    for n in declared_functions():
        if n in ("tt_status_string", "tt_last_error_message", "tt_version"):
            continue
        assert hasattr(tt, n), n


def test_status_strings(lib):
    lib.tt_status_string.restype = ctypes.c_char_p
    assert lib.tt_status_string(0) == b"TT_OK"
    assert lib.tt_status_string(4) == b"TT_ERR_WORKSPACE"
    lib.tt_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.tt_version()


def test_validation_errors_without_gpu(lib):
    i64, p, sz = ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
    f = lib.tt_local_matvec
    f.argtypes = [i64] * 5 + [p] * 6 + [sz, p]
    lib.tt_last_error_message.restype = ctypes.c_char_p
    fake = 4096
    assert f(0, 4, 1, 1, 1, fake, fake + 8, fake + 16, fake + 24, fake + 32, fake + 64, 10 ** 6, None) == 1
    assert f(1, 4, 1, 1, 1, None, fake, fake, fake, fake, fake, 10 ** 6, None) == 2
    assert f(1, 4, 1, 1, 1, fake, fake + 8, fake + 16, fake + 24, fake, fake + 64, 10 ** 6, None) == 3
    assert f(1, 4, 1, 1, 1, fake, fake + 8, fake + 16, fake + 24, fake + 32, None, 0, None) == 4
    assert b"workspace" in lib.tt_last_error_message()
    assert f(1 << 40, 1 << 20, 1 << 20, 1, 1, fake, fake + 8, fake + 16, fake + 24, fake + 32,
             fake + 64, 10 ** 6, None) == 5
    ws = lib.tt_local_matvec_workspace_size
    ws.argtypes = [i64] * 6
    ws.restype = sz
    assert ws(4, 4, 4, 2, 2, 1) > 0 and ws(0, 4, 4, 2, 2, 1) == 0
    # sweep: boundary ranks must be 1
    sw = lib.tt_sweep_interfaces
    sw.argtypes = [i64, p, p, p, p, p, p, p, ctypes.c_int, p, sz, p]
    n = (i64 * 2)(4, 4)
    r = (i64 * 3)(2, 3, 1)
    R = (i64 * 3)(1, 2, 1)
    arr = (p * 3)(fake, fake + 8, fake + 16)
    assert sw(2, n, r, R, arr, arr, arr, arr, 3, fake, 10 ** 6, None) == 1
    r = (i64 * 3)(1, 3, 1)
    assert sw(2, n, r, R, arr, arr, None, None, 7, fake, 10 ** 6, None) == 1


def test_no_oracle_in_product_path():
    """The product package never references the oracle (DESIGN.md §6 independence rule)."""
    pkg = os.path.join(ROOT, "paper_2509_11890_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                s = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in s.replace("no oracle", ""), fn


def _header_param_counts():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(tt_[a-z_0-9]+)\s*\(([^;{]*?)\)\s*;", src, flags=re.S):
        params = m.group(2).strip()
        out[m.group(1)] = 0 if params in ("", "void") else params.count(",") + 1
    return out


def test_binding_argtypes_match_header():
    """Every ctypes prototype of the binding has exactly the header's parameter count (a
    missing entry silently truncates a 64-bit argument, e.g. the stream)."""
    import paper_2509_11890_b200 as tt
    counts = _header_param_counts()
    checked = 0
    for name, n in counts.items():
        fn = getattr(tt.lib, name)
        if fn.argtypes is None:
            continue
        assert len(fn.argtypes) == n, (name, len(fn.argtypes), n)
        checked += 1
    assert checked >= 12


def test_debug_hooks_live_in_the_debug_header():
    """ABI hygiene: the production header declares no tt_debug_* hook; the debug header does."""
    prod = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    dbg = re.sub(r"/\*.*?\*/", "", open(DEBUG_HEADER).read(), flags=re.S)
    assert not re.findall(r"\btt_debug_[a-z_0-9]+\s*\(", prod)
    assert "tt_debug_set_flags" in dbg and "tt_debug_set_variant" in dbg


def test_product_library_reads_no_environment_knobs():
    """The probe knobs (TT_LAT_*, TT_PDL_FLOPS, TT_L2_DEBUG) exist only in a debug build."""
    data = open(LIB, "rb").read()
    for knob in (b"TT_LAT_FLOPS", b"TT_PDL_FLOPS", b"TT_L2_DEBUG", b"TT_LAT_UNIT_US"):
        assert knob not in data, knob


def test_matvec_mode_sizes_the_workspace(lib):
    """tt_set_matvec_mode (host logic only): an unknown mode is rejected; under TT_MATVEC_FUSED
    the workspace of an eligible core drops T1 = rl Rl n nvec rr doubles, an ineligible core
    (n != 4, rr % 16 != 0, Rr % 4 != 0, Rl > 36, odd rl) keeps it; AUTO restores the size."""
    import ctypes
    f = lib.tt_local_matvec_workspace_size
    f.restype = ctypes.c_size_t
    f.argtypes = [ctypes.c_int64] * 6
    lib.tt_set_matvec_mode.restype = ctypes.c_int
    lib.tt_set_matvec_mode.argtypes = [ctypes.c_int]
    assert lib.tt_set_matvec_mode(7) != 0
    elig = (256, 4, 256, 36, 36, 32)
    inelig = [(256, 3, 256, 36, 36, 32), (256, 4, 250, 36, 36, 32), (256, 4, 256, 36, 35, 32),
              (256, 4, 256, 40, 36, 32), (255, 4, 256, 36, 36, 32)]
    full = f(*elig)
    full_in = [f(*s) for s in inelig]
    assert lib.tt_set_matvec_mode(2) == 0
    try:
        t1 = 8 * 256 * 36 * 4 * 32 * 256
        assert full - t1 - 4096 <= f(*elig) <= full - t1
        assert [f(*s) for s in inelig] == full_in
    finally:
        assert lib.tt_set_matvec_mode(0) == 0
    assert f(*elig) == full
