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
    assert abs(eps3) <= 1e-12 * eps2


@pytest.mark.parametrize("name,N1,N2,tol2", [("c4", 4, 8, 1e-5), ("c5", 3, 4, 2e-2)])
def test_tgv_initial_strain_dissipation_converges(name, N1, N2, tol2):
    (_, e1, _), mu = _diag(name, N1)
    (_, e2, _), _ = _diag(name, N2)
    exact = 2.0 * mu * 3.0 / 8.0
    err1, err2 = abs(e1 - exact) / exact, abs(e2 - exact) / exact
    assert err2 < tol2 and err2 < err1 / 3.0, (err1, err2)
