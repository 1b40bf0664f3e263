"""C-ABI library on the CPU: exports, host setup (operators, meshes) vs the oracle.

No GPU compute calls here.  Operators are built independently (product: C++
__float128, closed-form tensor factors / shifted-monomial simplex Vandermonde;
oracle: 40-digit monomial Vandermonde), so agreement to ~1 ulp is a real check.
Integer maps must agree bit-exactly (BASELINE.json north_star).
"""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle.mesh import build_mesh
from oracle.operators import build_operators

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sdrt():
    from paper_2105_08632_b200.build import build
    build()
    from paper_2105_08632_b200 import sdrt as S
    return S


def test_library_exports_every_header_symbol(sdrt):
    hdr = open(os.path.join(ROOT, "include", "sdrt.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)          # strip comments
    names = set(re.findall(r"\b(sdrt_[a-z_]+)\s*\(", hdr))
    assert len(names) >= 15
    lib = ctypes.CDLL(sdrt._LIBPATH)
    for n in sorted(names):
        assert hasattr(lib, n), n
    assert set(sdrt.EXPORTED) <= names
    assert sdrt.abi_version() == 1


CASES = [("quad", 1), ("quad", 2), ("quad", 3), ("quad", 4), ("tri", 1), ("tri", 2), ("tri", 3),
         ("tri", 4), ("hex", 1), ("hex", 2), ("hex", 3), ("hex", 4), ("tet", 1), ("tet", 2), ("tet", 3),
         ("pri", 1), ("pri", 2), ("pri", 3)]


@pytest.mark.parametrize("etype,p", CASES)
def test_operators_match_oracle(sdrt, etype, p):
    o = sdrt.operators_build(etype, p)
    O = build_operators(etype, p)
    try:
        for nm in ["M0", "M12", "M13", "M14", "M15", "M16", "P", "M19P2"]:
            A = sdrt.operators_get(o, nm)
            B = getattr(O, nm)
            assert A.shape == B.shape, nm
            assert np.abs(A - B).max() <= 4e-16 * max(1.0, np.abs(B).max()), nm
        w = sdrt.operators_get(o, "w")[:, 0]
        assert np.abs(w - O.w).max() < 1e-15
        for nm, ref in [("xsol", O.xsol), ("xext", O.xext), ("xu", O.xu)]:
            assert np.abs(sdrt.operators_get(o, nm) - ref).max() < 1e-15
    finally:
        sdrt.operators_destroy(o)


@pytest.mark.parametrize("etype,p,N", [("quad", 2, 3), ("quad", 2, (4, 3)), ("tri", 3, 4), ("hex", 1, 3),
                                       ("hex", 3, (3, 4, 5)), ("tet", 1, 3), ("tet", 3, 4), ("pri", 2, (3, 4, 3)),
                                       ("pri", 3, 3)])
def test_mesh_maps_bit_exact(sdrt, etype, p, N):
    D = 2 if etype in ("quad", "tri") else 3
    Nl = list(N) if isinstance(N, tuple) else [N] * D
    lo, hi = [0.0] * D, [1.0 + 0.5 * d for d in range(D)]
    m = sdrt.mesh_create(etype, p, Nl, lo, hi)
    try:
        fe, fl, fp, il = sdrt.mesh_export_maps(m)
        M = build_mesh(etype, p, tuple(Nl), lo, hi)
        assert fe.dtype == np.int32 and np.array_equal(fe, M.face_elem)
        assert np.array_equal(fl, M.face_lface)
        assert np.array_equal(fp, M.face_perm)
        assert np.array_equal(il.astype(bool), M.is_left)
        assert np.abs(sdrt.mesh_sol_coords(m) - M.sol_coords()).max() < 1e-14
        assert np.allclose(sdrt.mesh_detj(m), M.detJ, rtol=1e-15, atol=0)
    finally:
        sdrt.mesh_destroy(m)


@pytest.mark.parametrize("etype,p,N,per", [("quad", 2, (4, 3), (0, 1)), ("tri", 3, (4, 3), (0, 1)),
                                           ("hex", 2, (3, 4, 3), (0, 1, 1)), ("tet", 2, (3, 3, 4), (1, 0, 1)),
                                           ("pri", 2, (3, 3, 4), (1, 1, 0))])
def test_farfield_mesh_maps_bit_exact(sdrt, etype, p, N, per):
    """Far-field meshes (non-periodic axis): the face list (boundary
    faces with -1 for the exterior side) and the left flags equal the oracle's."""
    D = len(N)
    lo, hi = [0.0] * D, [1.0 + 0.5 * d for d in range(D)]
    m = sdrt.mesh_create(etype, p, list(N), lo, hi, periodic=per)
    try:
        fe, fl, fp, il = sdrt.mesh_export_maps(m)
        M = build_mesh(etype, p, tuple(N), lo, hi, periodic=per)
        assert (fe < 0).any()
        assert np.array_equal(fe, M.face_elem)
        assert np.array_equal(fl, M.face_lface)
        assert np.array_equal(fp, M.face_perm)
        assert np.array_equal(il.astype(bool), M.is_left)
    finally:
        sdrt.mesh_destroy(m)


def test_errors_are_reported(sdrt):
    with pytest.raises(sdrt.SdrtError) as e:
        sdrt.operators_build("tet", 4)
    assert e.value.code == -2
    with pytest.raises(sdrt.SdrtError) as e:
        sdrt.mesh_create("quad", 2, [2, 2], [0, 0], [1, 1])
    assert e.value.code == -1
    with pytest.raises(sdrt.SdrtError) as e:
        sdrt.operators_build("quad", 0)
    assert e.value.code == -2


def test_fr_schemes_build(sdrt):
    """FR-SDRT and FR-DG build for every element type; the SDRT scheme has no "Mc"."""
    for sch in ("frsdrt", "frdg"):
        for et in ("quad", "tri", "hex", "tet"):
            o = sdrt.operators_build(et, 2, sch)
            assert sdrt.operators_get(o, "Mc").shape == sdrt.operators_get(o, "M14").shape
            sdrt.operators_destroy(o)
    o = sdrt.operators_build("tri", 2)
    with pytest.raises(sdrt.SdrtError):
        sdrt.operators_get(o, "Mc")
    sdrt.operators_destroy(o)


@pytest.mark.parametrize("etype,p", [c for c in CASES if c[0] != "pri"])
def test_fr_corrections_match_oracle(sdrt, etype, p):
    """Mc of the library (collapsed Gauss quadrature in __float128 for the simplex DG
    lifting) against the oracle (exact monomial integrals; Radau on tensor elements)."""
    from oracle.fr import dg_correction_tensor, dg_lift
    for sch, ref in (("frsdrt", build_operators(etype, p).M14),
                     ("frdg", dg_correction_tensor(etype, p) if etype in ("quad", "hex") else dg_lift(etype, p))):
        o = sdrt.operators_build(etype, p, sch)
        try:
            A = sdrt.operators_get(o, "Mc")
            assert np.abs(A - ref).max() <= 1e-14 * np.abs(ref).max(), (sch, np.abs(A - ref).max())
        finally:
            sdrt.operators_destroy(o)
