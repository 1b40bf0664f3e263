"""TGV diagnostics (NEXT row N4): oracle pins against closed forms
of the Taylor-Green initial field (no GPU).

For v = (sin x cos y cos z, -cos x sin y cos z, 0) on [0, 2 pi]^3:
  <v.v> = 1/4 and the density perturbation of the initial pressure field integrates
  against v.v to zero, so <E*> = <rho v.v> = 1/4;  div v = 0, so S^d = S and
  <S : S> = 3/8 (integrals of products of sines and cosines), eps2 = 2 mu 3/8, eps3 = 0.
The discrete values use the LDG gradient of the collocated initial field, so eps2
converges to 3 mu / 4 with the mesh (design order), while <E*> and eps3 hold to round-off.
"""
import math

import pytest

from oracle.diagnostics import tgv_diagnostics
from oracle.mesh import build_mesh
from oracle.physics import Physics
from oracle.residual import Residual
from sdrt_inputs import CONFIGS, initial_state, scaled


def _diag(name, N):
    c = scaled(CONFIGS[name], N)
    m = build_mesh(c.etype, c.p, N, c.lo, c.hi)
    R = Residual(m, Physics("ns", 3, **c.physics_kwargs()))
    return tgv_diagnostics(R, initial_state(c, m.sol_coords())), c.physics_kwargs()["mu"]


@pytest.mark.parametrize("name,N", [("c4", 4), ("c5", 3)])
def test_tgv_initial_energy_and_pressure_dissipation(name, N):
    (E, eps2, eps3), mu = _diag(name, N)
    assert abs(E - 0.25) <= 1e-12
    # eps3 = -<p div v> with div v = 0: round-off of an integrand p (~p_inf = 71.4) times
    # a unit-size gradient, so the scale is p_inf, not eps2 (~mu = 1/1600)
    pinf = 1.0 / (1.4 * 0.1 ** 2)
    assert abs(eps3) <= 1e-13 * pinf


@pytest.mark.parametrize("name,N1,N2,tol2", [("c4", 4, 8, 1e-5), ("c5", 3, 4, 2e-2)])
def test_tgv_initial_strain_dissipation_converges(name, N1, N2, tol2):
    (_, e1, _), mu = _diag(name, N1)
    (_, e2, _), _ = _diag(name, N2)
    exact = 2.0 * mu * 3.0 / 8.0
    err1, err2 = abs(e1 - exact) / exact, abs(e2 - exact) / exact
    assert err2 < tol2 and err2 < err1 / 3.0, (err1, err2)


# ---------------------------------------------------------------- degree-10 quadrature (l.2075)
import itertools

import numpy as np

from oracle.diagnostics import cubature
from oracle.operators import _mono_integral


@pytest.mark.parametrize("etype", ["quad", "tri", "hex", "tet"])
@pytest.mark.parametrize("degree", [2, 5, 10])
def test_cubature_exact_to_degree(etype, degree):
    """The rule integrates every monomial of total degree <= degree exactly (against the
    closed-form monomial integrals of the reference element), and its weights sum to the
    reference volume."""
    D = 2 if etype in ("quad", "tri") else 3
    x, w, _ = cubature(etype, degree)
    for e in itertools.product(range(degree + 1), repeat=D):
        if sum(e) > degree:
            continue
        ex = float(_mono_integral(etype, e))
        assert abs((w * np.prod(x ** np.array(e), axis=1)).sum() - ex) <= 1e-14, e
    assert (w > 0).all()


@pytest.mark.parametrize("name,N,p", [("c4", 3, 3), ("c5", 2, 2)])
def test_cubature_integrates_polynomial_integrands_exactly(name, N, p):
    """Constant density: E* (degree 2p), S^d:S^d (2p) and p div v (3p <= 10) of the
    interpolated fields are polynomials, so the degree-10 rule and a degree-14 rule agree
    to round-off (a wrong interpolation matrix or weight would not)."""
    from dataclasses import replace
    c = replace(scaled(CONFIGS[name], N), p=p)
    m = build_mesh(c.etype, p, N, c.lo, c.hi)
    R = Residual(m, Physics("ns", 3, **c.physics_kwargs()))
    from sdrt_inputs import random_state
    U = random_state(c, R.ops.nsol, m.K, seed=4, amp=0.3)
    U[:, 0, :] = 1.3
    a = np.array(tgv_diagnostics(R, U, 10))
    b = np.array(tgv_diagnostics(R, U, 14))
    assert (np.abs(a - b) <= 1e-12 * np.abs(b).max()).all(), (a, b)
    s = np.array(tgv_diagnostics(R, U))
    assert np.abs(s - b).max() > 1e-8 * np.abs(b).max()     # the solution-point sums differ


@pytest.mark.parametrize("name,N1,N2,ratio", [("c4", 4, 8, 50.0), ("c5", 3, 4, 2.0)])
def test_tgv_cubature_energy_converges(name, N1, N2, ratio):
    """<E*> of the collocated initial field by the degree-10 rule converges to 1/4 (the
    interpolant of rho v.v is not exact, unlike the solution-point sum)."""
    def run(N):
        c = scaled(CONFIGS[name], N)
        m = build_mesh(c.etype, c.p, N, c.lo, c.hi)
        R = Residual(m, Physics("ns", 3, **c.physics_kwargs()))
        E, e2, e3 = tgv_diagnostics(R, initial_state(c, m.sol_coords()), 10)
        return abs(E - 0.25), e2
    err1, _ = run(N1)
    err2, _ = run(N2)
    assert err2 < err1 / ratio and err2 < 1e-3, (err1, err2)
