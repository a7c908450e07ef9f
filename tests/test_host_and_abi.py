"""CPU-side checks of the product library: it loads, exports every symbol
include/sait_c.h declares, and its host input producers (ILU(k), generators)
are bitwise identical to the oracle's."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from helpers import bitwise_equal, bitwise_equal_csr, to_product


def header_functions():
    src = open(os.path.join(ROOT, "include", "sait_c.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sait_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import ctypes

    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2106_12836_b200", "libsait_b200.so"))
    names = header_functions()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2106_12836_b200 import _native as N

    assert set(header_functions()) == set(N.PROTOTYPES), set(header_functions()) ^ set(N.PROTOTYPES)
    assert N.lib.sait_abi_version() == 1


def test_generators_match_oracle():
    import paper_2106_12836_b200 as S
    from oracle import oracle as O

    assert bitwise_equal_csr(S.laplacian_2d(37), O.laplacian_2d(37))
    assert bitwise_equal_csr(S.laplacian_3d(11), O.laplacian_3d(11))
    assert bitwise_equal_csr(S.convdiff_2d(45), O.convdiff_2d(45))
    assert bitwise_equal_csr(S.convdiff_2d(17, -3.0, 4.0), O.convdiff_2d(17, -3.0, 4.0))
    assert bitwise_equal_csr(S.synthetic_lower(5000), O.synthetic_lower(5000))
    assert bitwise_equal(S.uniform_pm1(1234, 777), O.uniform_pm1(1234, 777))
    A = S.laplacian_3d(128)
    assert A.nnz() == 14581760  # 7 n^3 - 6 n^2
    assert S.laplacian_2d(64).nnz() == 20224


@pytest.mark.parametrize("level", [0, 1, 2])
def test_ilu_matches_oracle(port, level):
    import paper_2106_12836_b200 as S
    from oracle import oracle as O

    for A in (O.laplacian_3d(10), O.convdiff_2d(25), O.laplacian_2d(30)):
        L, U = port.ilu_k(A, level)
        f = S.ilu_k(to_product(A), level)
        assert bitwise_equal_csr(f.lower, L) and bitwise_equal_csr(f.upper, U)


def test_ilu_errors():
    import paper_2106_12836_b200 as S

    a = S.CsrMatrix(2, 2, [0, 1, 2], [1, 0], [1.0, 1.0])
    with pytest.raises(S.SaitInvalidArgument, match="ilu_k: structurally zero diagonal at row 0"):
        S.ilu_k(a, 0)
    z = S.CsrMatrix(2, 2, [0, 2, 4], [0, 1, 0, 1], [1.0, 1.0, 1.0, 1.0])
    with pytest.raises(S.SaitRuntimeError, match="ilu_k: pivot breakdown at row 1"):
        S.ilu_k(z, 0)


def test_synthetic_config4_shape():
    import paper_2106_12836_b200 as S

    t = S.synthetic_lower(200000)
    per_row = t.nnz() / t.nrows
    assert 15.0 < per_row < 16.0  # ~15.5 incl. diagonal
    diag = t.values[t.row_ptr[1:] - 1]
    off = np.abs(t.values).sum() - np.abs(diag).sum()
    assert np.allclose(diag.sum(), 1.5 * off + t.nrows)


STRUCTS = [("sait_host_csr", "HostCsr"), ("sait_drop_spec", "DropSpec"), ("sait_build_stats", "BuildStats"),
           ("sait_solve_stats", "SolveStats"), ("sait_row_piece", "RowPiece"), ("sait_halo_t", "Halo"),
           ("sait_peer_factor_desc", "PeerFactorDesc"), ("sait_factor_format", "FactorFormat")]


def test_ctypes_structs_match_header(tmp_path):
    """The ctypes mirrors of the C ABI's structs have the header's size and
    field offsets (a C program compiled against include/sait_c.h prints
    them)."""
    import ctypes
    import shutil
    import subprocess

    from paper_2106_12836_b200 import _native as N

    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "sait_c.h"', "int main(void) {"]
    for cname, pyname in STRUCTS:
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in getattr(N, pyname)._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("  return 0;\n}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    inc = os.path.join(ROOT, "include")
    subprocess.run(["gcc", "-I", inc, "-I/usr/local/cuda/include", str(src), "-o", str(exe)], check=True)
    got = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    for cname, pyname in STRUCTS:
        cls = getattr(N, pyname)
        assert f"{cname} size {ctypes.sizeof(cls)}" in got, cname
        for fname, _ in cls._fields_:
            assert f"{cname} {fname} {getattr(cls, fname).offset}" in got, (cname, fname)
