"""CPU: the C-ABI library loads and exports every entry point include/pit_b200.h declares.

No compute calls are made here (no GPU in the build container); only argument validation paths
that return before touching the device.
"""

import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "pit_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"PIT_API\s+[\w\s\*]+?\b(pit_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2301_10936_b200 import _lib

    return _lib.load()


def test_header_declares_the_reference_boundary():
    syms = declared_symbols()
    for want in ("pit_build_index", "pit_build_index_from_tensor", "pit_sread", "pit_swrite", "pit_spmm",
                 "pit_last_error"):
        assert want in syms


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_python_binding_covers_every_symbol():
    from paper_2301_10936_b200 import _lib

    assert sorted(_lib.EXPORTS) == declared_symbols()


def test_geometry_and_validation_without_gpu(lib):
    from paper_2301_10936_b200 import _lib

    ng, pg, wg = C.c_int64(), C.c_int64(), C.c_int64()
    assert lib.pit_index_geometry(1024, 1024, 32, 1, 1, C.byref(ng), C.byref(pg), C.byref(wg)) == _lib.PIT_OK
    assert (ng.value, pg.value, wg.value) == (32, 1024, 32)
    assert lib.pit_index_geometry(45, 70, 1, 32, 0, C.byref(ng), C.byref(pg), C.byref(wg)) == _lib.PIT_OK
    assert (ng.value, pg.value, wg.value) == (3, 45, 2)
    assert lib.pit_index_geometry(4, 4, 0, 2, 0, C.byref(ng), C.byref(pg), C.byref(wg)) == _lib.PIT_ERR_ARG
    assert "positive" in _lib.last_error()
    assert lib.pit_index_geometry(4, 4, 1, 2, 3, C.byref(ng), C.byref(pg), C.byref(wg)) == _lib.PIT_ERR_ARG
    args = _lib.SpmmArgs()
    args.plan = 9
    assert lib.pit_spmm(C.byref(args), None) == _lib.PIT_ERR_ARG
    args.plan = _lib.PIT_PLAN_PIT_K
    args.dtype = _lib.PIT_BF16
    args.M = args.N = args.K = 64
    args.A = args.B = args.C = 16
    args.sam, args.sak = 64, 1
    assert lib.pit_spmm(C.byref(args), None) == _lib.PIT_ERR_LAYOUT
    assert "col_major" in _lib.last_error()
    assert lib.pit_abi_version() == 104
    assert lib.pit_kernel_launches() == 0


def test_workspace_query_without_gpu(lib):
    """pit_spmm_workspace_bytes is a host-only query: scratch only for the split gathered-K case (few
    128-row groups, N <= 64), none for C1-style launches or the CUDA-core path."""
    from paper_2301_10936_b200 import _lib

    def args(t0, n, groups):
        a = _lib.SpmmArgs()
        a.plan, a.dtype = _lib.PIT_PLAN_PIT_K, _lib.PIT_BF16
        a.M, a.N, a.K = groups * t0, n, 4096
        a.A = a.B = a.C = 1 << 20  # aligned placeholders: never dereferenced
        a.sam, a.sak, a.ldb, a.ldc = 1, groups * t0, n, n
        a.t0, a.t1, a.n_groups, a.slot_stride = t0, 1, groups, 4096
        return a

    attn = args(128, 64, 384)
    assert lib.pit_spmm_workspace_bytes(C.byref(attn)) > 0
    assert lib.pit_spmm_workspace_bytes(C.byref(args(128, 8192, 384))) == 0
    assert lib.pit_spmm_workspace_bytes(C.byref(args(32, 64, 384))) == 0
    attn.force_simt = 1
    assert lib.pit_spmm_workspace_bytes(C.byref(attn)) == 0


def test_spmm_args_struct_matches_header():
    """Field order of the ctypes mirror equals the C struct's."""
    from paper_2301_10936_b200 import _lib

    import re

    body = HEADER.read_text().split("typedef struct {", 1)[1].split("} pit_spmm_args;", 1)[0]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = []
    for line in body.splitlines():
        line = line.split("/*")[0].strip().rstrip(";")
        if not line:
            continue
        decl = line.split(None, 1)[1] if not line.startswith("const") else line.split(None, 2)[2]
        for part in decl.split(","):
            names.append(part.replace("*", "").strip())
    assert names == [f[0] for f in _lib.SpmmArgs._fields_]
