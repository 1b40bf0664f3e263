"""Pins of the oracle FR-SDRT / FR-DG residuals (NEXT row N1; no GPU).

* FR-SDRT == SDRT for linear flux on constant-metric elements (§2.3,
  Eq. divergence_equivalence l.414-419 and the gradient remark l.429-434; the paper's
  runs agree to 6.11e-16, Tables l.1855, l.1866), on every element type.
* FR-DG on quadrilaterals reproduces the paper's FR-DG tau_MAX tables (advection
  l.1236-1243, diffusion l.1576-1585) with the oracle's Von Neumann harness.
* FR-DG on simplices (the DG lifting, oracle.fr.dg_lift): equals the Radau form on
  tensor elements (two independent constructions of the same correction), integrates
  to the face measure, and reproduces the paper's FR-DG triangle tau_MAX tables
  (diffusion l.1612-1618; advection l.1255, l.1272 through the FR-DG/SDRT ratio, since the
  simplex advection length scale differs by a constant factor).
* freestream and discrete conservation for both schemes (l.170-172, l.312-318).
"""
import functools

import numpy as np
import pytest

from oracle import vonneumann as VN
from oracle.fr import FRResidual, dg_correction_tensor, dg_lift
from oracle.mesh import build_mesh
from oracle.operators import build_operators
from oracle.physics import Physics
from oracle.residual import Residual
from sdrt_inputs import CONFIGS, random_state

import json
import os

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_tables.json")))
ND = {"quad": 2, "tri": 2, "hex": 3, "tet": 3}


@pytest.mark.parametrize("etype,p,N", [("quad", 3, 4), ("tri", 3, 3), ("hex", 2, 2), ("tet", 2, 2), ("tet", 3, 2)])
def test_frsdrt_equals_sdrt_linear(etype, p, N):
    D = ND[etype]
    m = build_mesh(etype, p, N, [0.0] * D, [1.0] * D)
    ph = Physics("linadvdiff", D, c=tuple([1.0, 0.6, 0.3][:D]), mu=0.05)
    U = np.random.default_rng(1).uniform(-1, 1, (build_operators(etype, p).nsol, 1, m.K))
    a, b = Residual(m, ph)(U), FRResidual(m, ph, "frsdrt")(U)
    assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()


def test_frsdrt_differs_from_sdrt_nonlinear():
    """Non-linear flux: the schemes differ (aliasing, l.386-389) - the equivalence above is
    not a tautology of the implementation."""
    cfg = CONFIGS["c2"]
    m = build_mesh("tri", 3, 3, cfg.lo, cfg.hi)
    ph = Physics("euler", 2, **cfg.physics_kwargs())
    U = random_state(cfg, build_operators("tri", 3).nsol, m.K, seed=5, amp=0.3)
    a, b = Residual(m, ph)(U), FRResidual(m, ph, "frsdrt")(U)
    assert np.abs(a - b).max() > 1e-8 * np.abs(a).max()


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_frdg_quad_tau_max_tables(p):
    res = functools.partial(FRResidual, scheme="frdg")
    B = VN.pattern_blocks("quad", p, VN.diffusion_physics(2), layers=2, residual=res)
    lam = VN.spectrum(B, [np.array([k, 0.0]) for k in np.linspace(0, 2 * np.pi, 361)])
    assert lam.real.max() < 1e-10
    ref = GOLD["tau_max_frdg_quad"]["diffusion"][str(p)]
    for stages, r in zip((3, 4, "rk54"), ref):
        assert abs(VN.tau_max(lam, stages) - r) <= 1.5e-4, (stages, VN.tau_max(lam, stages), r)
    ph = VN.advection_physics(2)
    d = np.array(ph.c)
    B = VN.pattern_blocks("quad", p, ph, layers=1, residual=res)
    lam = VN.spectrum(B, [k * d for k in np.linspace(0, np.pi / np.abs(d).max(), 401)])
    assert abs(VN.tau_max(lam, 4) - GOLD["tau_max_frdg_quad"]["advection"][str(p)][1]) <= 2.5e-3


@pytest.mark.parametrize("etype,p", [("quad", 1), ("quad", 2), ("quad", 3), ("quad", 4), ("hex", 1), ("hex", 2)])
def test_dg_lift_equals_radau_on_tensor(etype, p):
    """The generic DG lifting (mass matrix + face integrals) and Huynh's Radau g_DG are
    built by unrelated formulas; on tensor elements they are the same correction."""
    a, b = dg_lift(etype, p), dg_correction_tensor(etype, p)
    assert np.abs(a - b).max() <= 1e-14 * np.abs(b).max()


@pytest.mark.parametrize("etype,p", [("tri", 1), ("tri", 2), ("tri", 3), ("tri", 4), ("tet", 1), ("tet", 2)])
def test_dg_lift_face_measure(etype, p):
    """sum_s w_s div g_nu(x_s) = int div g_nu = int_face ell_nu dS: the face weights, which
    sum to the face measure (tri: 2, 2 sqrt2, 2; tet: 2, 2, 2 sqrt3, 2), and the lifted
    correction of a face's constant is the same for every point ordering."""
    o = build_operators(etype, p)
    fw = o.w @ dg_lift(etype, p)
    area = {"tri": [2, 2 * np.sqrt(2), 2], "tet": [2, 2, 2 * np.sqrt(3), 2]}[etype]
    for f in range(o.nfaces):
        assert abs(fw[o.ext_face == f].sum() - area[f]) <= 1e-13
    assert (fw > 0).all()


GOLD_FRDG_TRI = {  # FR-DG Triangles, diffusion tau_MAX (RK3, RK4, RK54)
    1: [0.0418, 0.0464, 0.0776], 2: [0.0144, 0.0160, 0.0267], 3: [0.0054, 0.0060, 0.0101], 4: [0.0027, 0.0030, 0.0050]}


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_frdg_tri_tau_max_tables(p):
    res = functools.partial(FRResidual, scheme="frdg")
    B = VN.pattern_blocks("tri", p, VN.diffusion_physics(2), layers=2, residual=res)
    lam = VN.spectrum(B, [np.array([k, 0.0]) for k in np.linspace(0, 2 * np.pi, 361)])
    assert lam.real.max() < 1e-10
    for stages, r in zip((3, 4, "rk54"), GOLD_FRDG_TRI[p]):
        assert abs(VN.tau_max(lam, stages) - r) <= 1.2e-4, (stages, VN.tau_max(lam, stages), r)


def test_frdg_tri_advection_ratio():
    """Advection, triangles p=2, RK4: FR-DG / SDRT = 0.140 / 0.198 (l.1272, l.1255)."""
    ph = VN.advection_physics(2)
    d = np.array(ph.c)
    ks = [k * d for k in np.linspace(0, np.pi / np.abs(d).max(), 401)]
    t = {}
    for name, res in (("sdrt", Residual), ("frdg", functools.partial(FRResidual, scheme="frdg"))):
        lam = VN.spectrum(VN.pattern_blocks("tri", 2, ph, layers=1, residual=res), ks)
        t[name] = VN.tau_max(lam, 4)
    assert abs(t["frdg"] / t["sdrt"] - 0.140 / 0.198) <= 0.01, t


@pytest.mark.parametrize("p,ratio", [(1, 0.138 / 0.172), (2, 0.095 / 0.124)])
def test_frdg_tet_advection_ratio(p, ratio):
    """Advection on tetrahedra (theta0 = pi/6, theta1 = pi/4), RK4: FR-DG stays spatially
    stable and its tau_MAX relative to SDRT matches the paper's tables (SDRT Tetrahedra
    l.1329-1330, FR-DG Tetrahedra l.1346-1347; the absolute simplex values differ by a
    length-scale factor) within 0.02 (kappa sampled along c only)."""
    ph = VN.advection_physics(3)
    d = np.array(ph.c)
    ks = [k * d for k in np.linspace(0, np.pi / np.abs(d).max(), 201)]
    t = {}
    for name, res in (("sdrt", Residual), ("frdg", functools.partial(FRResidual, scheme="frdg"))):
        lam = VN.spectrum(VN.pattern_blocks("tet", p, ph, layers=1, residual=res), ks)
        assert lam.real.max() < 1e-12
        t[name] = VN.tau_max(lam, 4)
    assert abs(t["frdg"] / t["sdrt"] - ratio) <= 0.02, t


@pytest.mark.parametrize("scheme,etype,p", [("frsdrt", "tri", 3), ("frsdrt", "tet", 2), ("frsdrt", "hex", 2),
                                            ("frdg", "quad", 3), ("frdg", "hex", 2), ("frdg", "tri", 3),
                                            ("frdg", "tet", 2)])
def test_fr_freestream_and_conservation(scheme, etype, p):
    D = ND[etype]
    cfg = CONFIGS["c4" if D == 3 else "c2"]
    eq = "ns" if D == 3 else "euler"
    m = build_mesh(etype, p, 3, cfg.lo, cfg.hi)
    ph = Physics(eq, D, **cfg.physics_kwargs())
    R = FRResidual(m, ph, scheme)
    o = build_operators(etype, p)
    U = random_state(cfg, o.nsol, m.K, seed=2, amp=0.2)
    const = np.broadcast_to(U.mean(axis=(0, 2))[None, :, None], U.shape).copy()
    assert np.abs(R(const)).max() <= 1e-10 * np.abs(const).max()
    r = R(U)
    tot = np.einsum("r,rvk,k->v", o.w, r, m.detJ)
    mag = np.einsum("r,rvk,k->v", o.w, np.abs(r), m.detJ)
    assert (np.abs(tot) <= 1e-12 * mag).all(), (tot, mag)
