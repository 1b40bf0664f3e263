"""BASELINE.json configs c1..c5 and their initial conditions.

Readings: O15 (beta, eta per config), O16 (dt literals), O17 (Shu
vortex for c2), O18 (TGV units: rho_inf = v_inf = L = 1, p_inf = 1/(gamma Ma^2),
mu = 1/Re), O19 (domain [0, 2 pi]^3), O21 (nodal collocation of the IC), O23
(c3 Fourier modes, numpy default_rng(42)).
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field, replace

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    etype: str
    p: int
    N: int
    lo: tuple
    hi: tuple
    eq: str
    c: tuple = (0.0, 0.0, 0.0)
    mu: float = 0.0
    gamma: float = 1.4
    Pr: float = 0.71
    beta: float = 0.0
    eta: float = 0.0
    dt: float = 0.0
    steps: int = 0
    ic: str = ""
    nd: int = 2

    @property
    def nvars(self):
        return 1 if self.eq in ("linadv", "linadvdiff") else self.nd + 2

    @property
    def nsub(self):
        return {"quad": 1, "hex": 1, "tri": 2, "tet": 6, "pri": 2}[self.etype]

    @property
    def K(self):
        return self.N ** self.nd * self.nsub

    def physics_kwargs(self):
        return dict(c=self.c[: self.nd], mu=self.mu, gamma=self.gamma, Pr=self.Pr, beta=self.beta, eta=self.eta)


TGV_MA = 0.1
TGV_RE = 1600.0
TGV_PINF = 1.0 / (1.4 * TGV_MA ** 2)
_H4 = 2 * math.pi / 32
_H5 = 2 * math.pi / 48
_H3 = 2 * math.pi / 24

CONFIGS = {
    # c1: 2D linear advection, quads p=2, 8x8 on [0,1]^2, c=(1,1), dt=1e-3, 100 steps
    "c1": Config("c1", "quad", 2, 8, (0.0, 0.0), (1.0, 1.0), "linadv", c=(1.0, 1.0, 0.0),
                 dt=1e-3, steps=100, ic="sine2d", nd=2),
    # c2: 2D isentropic Euler vortex (Shu type, O17), 40x40 quads x 2 tris on [-5,5]^2, p=3,
    #     CFL 0.1 with h = 0.25 and lambda_max from the IC (tools/derive_dt.py, oracle only)
    "c2": Config("c2", "tri", 3, 40, (-5.0, -5.0), (5.0, 5.0), "euler", gamma=1.4,
                 dt=0.0, steps=1000, ic="vortex", nd=2),
    # c3: 3D linear advection-diffusion, hexes p=4, 24^3 on [0,2pi]^3, a=(1,1,1), nu=0.01,
    #     beta = eta = 0 (O15); dt = 2.5e-3 min(h/|a|, h^2/nu) (P:1798 rule)
    "c3": Config("c3", "hex", 4, 24, (0.0,) * 3, (2 * math.pi,) * 3, "linadvdiff", c=(1.0, 1.0, 1.0),
                 mu=0.01, beta=0.0, eta=0.0,
                 dt=2.5e-3 * min(_H3 / math.sqrt(3.0), _H3 ** 2 / 0.01), steps=200, ic="sines_modes", nd=3),
    # c4: TGV NS, hexes p=3, 32^3, Re=1600, Ma=0.1, Pr=0.71, beta=1/2, eta=0.1.
    #     dt = 0.06 h/11 (O16): the SURVEY's 0.1 h/11 is linearly unstable for Rusanov in 3D
    #     (measured: x0.9 and x0.75 of 0.1 h/11 diverge at steps 32 and 103; x0.6, x0.65
    #     run 500 steps); Rusanov applies the full |v.n|+c dissipation on all three axes,
    #     ~1.74x the per-axis load of the theta=(pi/6, pi/4) advection tau_MAX (0.131, l.1296)
    "c4": Config("c4", "hex", 3, 32, (0.0,) * 3, (2 * math.pi,) * 3, "ns", mu=1.0 / TGV_RE, gamma=1.4,
                 Pr=0.71, beta=0.5, eta=0.1, dt=0.06 * _H4 / 11.0, steps=500, ic="tgv", nd=3),
    # c5: TGV NS on tets p=3, 48^3 x 6 (663552 tets); dt = 0.035 h/11 (O16: 0.05 h/11
    #     diverges at step 169; x0.8 of it runs 200 steps; 0.7x taken for margin)
    "c5": Config("c5", "tet", 3, 48, (0.0,) * 3, (2 * math.pi,) * 3, "ns", mu=1.0 / TGV_RE, gamma=1.4,
                 Pr=0.71, beta=0.5, eta=0.1, dt=0.035 * _H5 / 11.0, steps=200, ic="tgv", nd=3),
}

# c4 on triangular prisms (NEXT row N3; PAPER.md's performance table covers prisms,
# l.2982-2995): same TGV, mesh 32^3 hexahedra x 2 prisms, p=3, c4's dt (a bench workload,
# not a BASELINE.json config)
CONFIGS["c4pri"] = replace(CONFIGS["c4"], name="c4pri", etype="pri")

# c2 dt literal: 0.1 * 0.25 / lambda_max, lambda_max = max(|v| + a) over the initial
# solution points (written by tools/derive_dt.py, which calls only oracle/)
C2_DT = 0.009923439617152275
CONFIGS["c2"] = replace(CONFIGS["c2"], dt=C2_DT)


def scaled(cfg: Config, N: int, steps: int | None = None) -> Config:
    """Same physics and dt on a smaller mesh (parity-test sizes)."""
    return replace(cfg, N=N, steps=cfg.steps if steps is None else steps)


def _conserved(rho, v, p, gamma):
    nd = len(v)
    U = np.empty((nd + 2,) + rho.shape)
    U[0] = rho
    for d in range(nd):
        U[1 + d] = rho * v[d]
    U[nd + 1] = p / (gamma - 1.0) + 0.5 * rho * sum(vi * vi for vi in v)
    return U


def c3_modes(seed=42):
    """O23: the 61 integer k with 0 < |k| <= 3, first non-zero component > 0,
    lexicographic order; phases from default_rng(seed)."""
    ks = []
    for k in itertools.product(range(-3, 4), repeat=3):
        if 0 < k[0] ** 2 + k[1] ** 2 + k[2] ** 2 <= 9:
            nz = [c for c in k if c != 0]
            if nz[0] > 0:
                ks.append(k)
    rng = np.random.default_rng(seed)
    ph = rng.uniform(0.0, 2 * np.pi, len(ks))
    return np.array(ks, dtype=np.float64), ph


def initial_state(cfg: Config, x: np.ndarray) -> np.ndarray:
    """IC at physical solution-point coordinates x of shape (N_sol, D, K) ->
    state (N_sol, N_V, K) (nodal collocation, O21)."""
    nsol, D, K = x.shape
    if cfg.ic == "sine2d":
        u = np.sin(2 * np.pi * x[:, 0]) * np.sin(2 * np.pi * x[:, 1])
        return u[:, None, :].copy()
    if cfg.ic == "sines_modes":
        u = np.sin(x[:, 0]) * np.sin(x[:, 1]) * np.sin(x[:, 2])
        ks, ph = c3_modes()
        for k, f in zip(ks, ph):
            u = u + 1e-2 * np.cos(k[0] * x[:, 0] + k[1] * x[:, 1] + k[2] * x[:, 2] + f)
        return u[:, None, :].copy()
    if cfg.ic == "vortex":
        g = cfg.gamma
        beta = 5.0
        uinf = 0.5 * math.sqrt(g)
        r2 = x[:, 0] ** 2 + x[:, 1] ** 2
        f = np.exp((1.0 - r2) / 2.0)
        u = uinf - beta / (2 * np.pi) * x[:, 1] * f
        v = beta / (2 * np.pi) * x[:, 0] * f
        T = 1.0 - (g - 1.0) * beta ** 2 / (8 * g * np.pi ** 2) * np.exp(1.0 - r2)
        rho = T ** (1.0 / (g - 1.0))
        p = rho ** g
        return np.moveaxis(_conserved(rho, [u, v], p, g), 0, 1).copy()
    if cfg.ic == "tgv":
        X, Y, Z = x[:, 0], x[:, 1], x[:, 2]
        v0 = np.sin(X) * np.cos(Y) * np.cos(Z)
        v1 = -np.cos(X) * np.sin(Y) * np.cos(Z)
        v2 = np.zeros_like(X)
        pinf = 1.0 / (cfg.gamma * TGV_MA ** 2)
        p = pinf + (1.0 / 16.0) * (np.cos(2 * X) + np.cos(2 * Y)) * (np.cos(2 * Z) + 2.0)
        rho = p / pinf
        return np.moveaxis(_conserved(rho, [v0, v1, v2], p, cfg.gamma), 0, 1).copy()
    raise ValueError(cfg.ic)


def random_state(cfg: Config, nsol: int, K: int, seed: int = 42, amp: float = 1.0) -> np.ndarray:
    """Seeded random state: linear U(-1,1); Euler/NS rho ~ U(0.8,1.2),
    v ~ U(-0.3,0.3) c_inf, p ~ U(0.8,1.2) p_inf (amp scales the spreads)."""
    rng = np.random.default_rng(seed)
    if cfg.nvars == 1:
        return rng.uniform(-1.0, 1.0, (nsol, 1, K))
    pinf = TGV_PINF if cfg.ic == "tgv" else 1.0
    cinf = math.sqrt(cfg.gamma * pinf)
    rho = 1.0 + amp * rng.uniform(-0.2, 0.2, (nsol, K))
    v = [amp * rng.uniform(-0.3, 0.3, (nsol, K)) * cinf for _ in range(cfg.nd)]
    p = pinf * (1.0 + amp * rng.uniform(-0.2, 0.2, (nsol, K)))
    return np.moveaxis(_conserved(rho, v, p, cfg.gamma), 0, 1).copy()
