"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no basis, no flux, no residual,
no estimator): only mesh connectivity and geometry nodes, per-element order
layouts, and the initial-condition formulas of BASELINE.json's configs
(``/root/repo/BASELINE.json`` configs[0..4]), evaluated at whatever node
coordinates the caller passes in.  Random numbers are drawn here once, with
``numpy.random.default_rng(seed)``, and handed identically to both sides.

Readings (DESIGN.md section "Input recipe"): A17, A20-A22 of SURVEY.md 8(c).2.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GAMMA = 1.4
BC_WALL = -1
BC_FARFIELD = -2

# Gauss-Lobatto node sets used to place GEOMETRY nodes (closed forms of the
# roots of (1-x^2)P_g'(x); mesh definition data, not the solver's basis).
_GEOM_NODES = {
    1: np.array([-1.0, 1.0]),
    2: np.array([-1.0, 0.0, 1.0]),
    3: np.array([-1.0, -1.0 / math.sqrt(5.0), 1.0 / math.sqrt(5.0), 1.0]),
    4: np.array([-1.0, -math.sqrt(3.0 / 7.0), 0.0, math.sqrt(3.0 / 7.0), 1.0]),
}


@dataclass
class Mesh:
    """Element connectivity + geometry-node coordinates.

    nbr[e, f]: element across face f = 2*d + s (d = xi/eta/zeta, s = 0 for the
    -1 side, 1 for the +1 side), or BC_WALL / BC_FARFIELD.
    geo[e, c, node]: coordinate c of geometry node (i,j,k) at the GL nodes of
    order gorder, node = i + (g1+1)*(j + (g2+1)*k).
    """

    nbr: np.ndarray
    gorder: tuple
    geo: np.ndarray
    dims: tuple = ()
    kind: str = "affine"
    extra: dict = field(default_factory=dict)

    @property
    def E(self) -> int:
        return int(self.nbr.shape[0])


def _lex(i, j, k, nx, ny):
    return i + nx * (j + ny * k)


def cube_mesh(nx: int, ny: int | None = None, nz: int | None = None, L=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0)) -> Mesh:
    """Periodic box [origin, origin+L] split into nx*ny*nz affine hexahedra,
    lexicographic element order (i fastest) [B:7-9]."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    E = nx * ny * nz
    nbr = np.empty((E, 6), np.int32)
    geo = np.empty((E, 3, 8), np.float64)
    h = (L[0] / nx, L[1] / ny, L[2] / nz)
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                e = _lex(i, j, k, nx, ny)
                nbr[e, 0] = _lex((i - 1) % nx, j, k, nx, ny)
                nbr[e, 1] = _lex((i + 1) % nx, j, k, nx, ny)
                nbr[e, 2] = _lex(i, (j - 1) % ny, k, nx, ny)
                nbr[e, 3] = _lex(i, (j + 1) % ny, k, nx, ny)
                nbr[e, 4] = _lex(i, j, (k - 1) % nz, nx, ny)
                nbr[e, 5] = _lex(i, j, (k + 1) % nz, nx, ny)
                for c, (ii, jj, kk) in enumerate([(a, b, cc) for cc in (0, 1) for b in (0, 1) for a in (0, 1)]):
                    geo[e, 0, c] = origin[0] + (i + ii) * h[0]
                    geo[e, 1, c] = origin[1] + (j + jj) * h[1]
                    geo[e, 2, c] = origin[2] + (k + kk) * h[2]
    return Mesh(nbr=nbr, gorder=(1, 1, 1), geo=geo, dims=(nx, ny, nz), kind="affine",
                extra={"h": h, "L": L})


def ogrid_mesh(nr: int, nth: int, nz: int, r0=0.5, r1=20.0, ratio=1.1, g_eta=4, Lz=1.0) -> Mesh:
    """Extruded O-grid around a unit-diameter cylinder (reading A22 / A21).

    Element (i, j, k): r in [r_i, r_{i+1}], r_i = r0 + dr0 (s^i - 1)/(s - 1),
    theta in [2 pi j/nth, 2 pi (j+1)/nth], z in [k, k+1] Lz/nz.  Local xi =
    radial outward (wall at xi=-1 of i=0, far field at xi=+1 of i=nr-1),
    eta = +theta, zeta = +z.  Geometry order (1, g_eta, 1): x,y = r(xi)
    (cos, sin)(theta(eta)) sampled at the GL nodes of order g_eta, so the
    geometry polynomial interpolates the arc; element order i fastest
    (radial), then azimuthal, then z.
    """
    s = ratio
    dr0 = (r1 - r0) * (s - 1.0) / (s ** nr - 1.0)
    radii = [r0 + dr0 * (s ** i - 1.0) / (s - 1.0) for i in range(nr + 1)]
    radii[-1] = r1
    E = nr * nth * nz
    ge = _GEOM_NODES[g_eta]
    ng = 2 * (g_eta + 1) * 2
    nbr = np.empty((E, 6), np.int32)
    geo = np.empty((E, 3, ng), np.float64)
    for k in range(nz):
        for j in range(nth):
            for i in range(nr):
                e = _lex(i, j, k, nr, nth)
                nbr[e, 0] = _lex(i - 1, j, k, nr, nth) if i > 0 else BC_WALL
                nbr[e, 1] = _lex(i + 1, j, k, nr, nth) if i < nr - 1 else BC_FARFIELD
                nbr[e, 2] = _lex(i, (j - 1) % nth, k, nr, nth)
                nbr[e, 3] = _lex(i, (j + 1) % nth, k, nr, nth)
                nbr[e, 4] = _lex(i, j, (k - 1) % nz, nr, nth)
                nbr[e, 5] = _lex(i, j, (k + 1) % nz, nr, nth)
                th0 = 2.0 * math.pi * j / nth
                th1 = 2.0 * math.pi * (j + 1) / nth
                for kk in range(2):
                    z = (k + kk) * Lz / nz
                    for jj in range(g_eta + 1):
                        th = th0 + 0.5 * (ge[jj] + 1.0) * (th1 - th0)
                        for ii in range(2):
                            r = radii[i + ii]
                            node = ii + 2 * (jj + (g_eta + 1) * kk)
                            geo[e, 0, node] = r * math.cos(th)
                            geo[e, 1, node] = r * math.sin(th)
                            geo[e, 2, node] = z
    return Mesh(nbr=nbr, gorder=(1, g_eta, 1), geo=geo, dims=(nr, nth, nz), kind="ogrid",
                extra={"radii": radii, "Lz": Lz})


def orders_uniform(E: int, N) -> np.ndarray:
    N = (N, N, N) if np.isscalar(N) else tuple(N)
    return np.tile(np.asarray(N, np.int32), (E, 1))


def orders_random(E: int, lo, hi, seed: int) -> np.ndarray:
    """i.i.d. uniform integer orders per element and direction, lo..hi inclusive
    (per-direction bounds allowed) [B:9, B:11]."""
    rng = np.random.default_rng(seed)
    lo = np.broadcast_to(np.asarray(lo), (3,))
    hi = np.broadcast_to(np.asarray(hi), (3,))
    out = np.empty((E, 3), np.int32)
    for d in range(3):
        out[:, d] = rng.integers(lo[d], hi[d] + 1, size=E)
    return out


def offsets(orders: np.ndarray, ncomp: int = 5) -> np.ndarray:
    n = np.prod(orders.astype(np.int64) + 1, axis=1)
    off = np.zeros(len(orders) + 1, np.int64)
    off[1:] = np.cumsum(ncomp * n)
    return off


def ndof(orders: np.ndarray) -> int:
    """NDOF = sum_e prod_d (N_d + 1)."""
    return int(np.prod(orders.astype(np.int64) + 1, axis=1).sum())


def conserved(rho, u, v, w, p, gamma=GAMMA):
    E = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v + w * w)
    return np.stack([rho, rho * u, rho * v, rho * w, E])


def pulse_state(X: np.ndarray, orders: np.ndarray, center=(0.5, 0.5, 0.5), sigma=0.1, amp=0.1,
                vel=(1.0, 0.5, 0.25), p=1.0, L=(1.0, 1.0, 1.0), gamma=GAMMA) -> np.ndarray:
    """Density pulse rho = 1 + amp exp(-d^2 / (2 sigma^2)), d the minimum-image
    (periodic) distance to the centre, u = vel, p const [B:7, reading A20].
    X: node coordinates in the canonical layout [e][3][n] (flattened)."""
    offx = offsets(orders, 3)
    offq = offsets(orders, 5)
    q = np.empty(offq[-1])
    for e in range(len(orders)):
        n = (offx[e + 1] - offx[e]) // 3
        x = X[offx[e]:offx[e + 1]].reshape(3, n)
        d2 = np.zeros(n)
        for c in range(3):
            dc = x[c] - center[c]
            dc = dc - L[c] * np.round(dc / L[c])
            d2 += dc * dc
        rho = 1.0 + amp * np.exp(-d2 / (2.0 * sigma * sigma))
        q[offq[e]:offq[e + 1]] = conserved(rho, vel[0] * np.ones(n), vel[1] * np.ones(n), vel[2] * np.ones(n),
                                          p * np.ones(n), gamma).ravel()
    return q


def uniform_state(orders: np.ndarray, rho=1.0, vel=(1.0, 0.5, 0.25), p=1.0, gamma=GAMMA) -> np.ndarray:
    offq = offsets(orders, 5)
    q = np.empty(offq[-1])
    qc = conserved(np.array(rho), np.array(vel[0]), np.array(vel[1]), np.array(vel[2]), np.array(p), gamma)
    for e in range(len(orders)):
        n = (offq[e + 1] - offq[e]) // 5
        q[offq[e]:offq[e + 1]] = np.repeat(qc, n)
    return q


def ns_params(Re=100.0, Ma=0.2, Pr=0.72, gamma=GAMMA):
    """Nondimensionalisation of reading A9: rho_inf = 1, |u_inf| = 1 along +x,
    D = 1, p_inf = 1/(gamma Ma^2), mu = 1/Re."""
    p_inf = 1.0 / (gamma * Ma * Ma)
    qinf = conserved(np.array(1.0), np.array(1.0), np.array(0.0), np.array(0.0), np.array(p_inf), gamma)
    return {"gamma": gamma, "mu": 1.0 / Re, "Pr": Pr, "qinf": np.asarray(qinf, np.float64), "p_inf": p_inf}


def freestream_noise_state(orders: np.ndarray, qinf_prims, noise=1e-3, seed=4, gamma=GAMMA) -> np.ndarray:
    """Free stream plus i.i.d. U(-1,1)*noise per velocity component per node,
    canonical order, rho = 1, p = p_inf (reading A22).  The draws are taken
    element by element, (3, n) per element (one vectorised draw of the same
    sequence)."""
    rho0, u0, v0, w0, p0 = qinf_prims
    rng = np.random.default_rng(seed)
    offq = offsets(orders, 5)
    n = np.diff(offq) // 5
    draws = rng.uniform(-1.0, 1.0, size=3 * int(n.sum())) * noise  # element e: 3 n_e values, [c][node]
    # per node: element, local node index -> positions of its u, v, w draws
    e_of = np.repeat(np.arange(len(n)), n)
    start = np.concatenate([[0], np.cumsum(3 * n)])[:-1]
    loc = np.arange(int(n.sum())) - np.repeat(np.concatenate([[0], np.cumsum(n)])[:-1], n)
    base = start[e_of] + loc
    du, dv, dw = draws[base], draws[base + n[e_of]], draws[base + 2 * n[e_of]]
    one = np.ones_like(du)
    Q = conserved(rho0 * one, u0 + du, v0 + dv, w0 + dw, p0 * one, gamma)  # [5][nodes]
    q = np.empty(offq[-1])
    qpos = np.repeat(offq[:-1], n) + loc
    for v in range(5):
        q[qpos + v * n[e_of]] = Q[v]
    return q


# --------------------------------------------------------------------------
# BASELINE.json configs (B:7-11) with the readings of SURVEY 8(c).2 / 8(d).
# --------------------------------------------------------------------------

def cfg2_center(seed=2):
    rng = np.random.default_rng(seed)
    return tuple(rng.uniform(0.3, 0.7, size=3))


CONFIGS = {
    "cfg1": dict(mesh=("cube", 4), orders=("uniform", 3), ic=dict(center=(0.5, 0.5, 0.5), sigma=0.1),
                 physics="euler", cfl=0.5, steps=10),
    "cfg2": dict(mesh=("cube", 16), orders=("uniform", 6), ic=dict(center="seed2", sigma=0.08),
                 physics="euler", cfl=0.5, tau_every=50, tau_max=1e-4, Nmin=3, Nmax=8),
    "cfg3": dict(mesh=("cube", 32), orders=("random", 2, 7, 3), ic=dict(center=(0.5, 0.5, 0.5), sigma=0.1),
                 physics="euler", cfl=0.5, steps=200, tau_every=20),
    "cfg4": dict(mesh=("ogrid", 48, 64, 1, 1.1, 4), orders=("uniform", 4), physics="ns", cfl=0.5),
    "cfg5": dict(mesh=("ogrid", 96, 256, 16, math.sqrt(1.1), 2), orders=("random_cfg5", 5), physics="ns", cfl=0.5),
}


def make_mesh(spec) -> Mesh:
    if spec[0] == "cube":
        return cube_mesh(spec[1])
    _, nr, nth, nz, ratio, g = spec
    return ogrid_mesh(nr, nth, nz, ratio=ratio, g_eta=g)


def make_orders(spec, E: int) -> np.ndarray:
    if spec[0] == "uniform":
        return orders_uniform(E, spec[1])
    if spec[0] == "random":
        return orders_random(E, spec[1], spec[2], spec[3])
    if spec[0] == "random_cfg5":  # reading A21: Nx, Ny ~ U{2..8}, Nz = 2
        return orders_random(E, (2, 2, 2), (8, 8, 2), spec[1])
    raise ValueError(spec)
