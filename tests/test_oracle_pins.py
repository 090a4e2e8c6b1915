"""Pins of the CPU oracle against what the paper and the mathematics fix
(SURVEY.md 8(c).3, Q1-Q16).  None of these re-types an oracle formula: each
checks a closed form, an invariant, a special case or a brute force.
"""
import json
import math
import os

import numpy as np
import pytest

import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _blocks(arr, orders, ncomp=5):
    off = W.offsets(orders, ncomp)
    for e in range(len(orders)):
        n = (off[e + 1] - off[e]) // ncomp
        yield e, arr[off[e]:off[e + 1]].reshape(ncomp, n)


# ----------------------------------------------------------------------------
# Q1 basis closed forms and quadrature exactness
# ----------------------------------------------------------------------------

def test_q1_gl_closed_forms(orc):
    g = json.load(open(os.path.join(GOLD, "gl_closed_forms.json")))
    for N, r in g["rules"].items():
        b = orc.basis(int(N))
        x = np.array([eval(s, {"sqrt": math.sqrt}) for s in r["x"]])
        w = np.array([eval(s, {"sqrt": math.sqrt}) for s in r["w"]])
        assert np.abs(b["x"] - x).max() < 1e-15
        assert np.abs(b["w"] - w).max() < 1e-15


@pytest.mark.parametrize("N", range(1, 13))
def test_q1_quadrature_exactness(orc, N):
    b = orc.basis(N)
    for k in range(0, 2 * N):  # GL is exact up to degree 2N-1
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs(np.sum(b["w"] * b["x"] ** k) - exact) < 1e-14
    # and NOT exact at degree 2N (it is a Lobatto rule, not Gauss)
    assert abs(np.sum(b["w"] * b["x"] ** (2 * N)) - 2.0 / (2 * N + 1)) > 1e-9


# ----------------------------------------------------------------------------
# Q2 D, D-hat, T, P
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("N", range(1, 10))
def test_q2_derivative_exact(orc, N):
    b = orc.basis(N)
    x = b["x"]
    for k in range(0, N + 1):
        d = b["D"] @ x ** k
        ref = k * x ** (k - 1) if k else np.zeros_like(x)
        assert np.abs(d - ref).max() < 1e-12 * max(1, N * N)
    # SBP / weak-form relation: W Dhat = -D^T W  (summation by parts)
    W_ = np.diag(b["w"])
    assert np.abs(W_ @ b["Dhat"] + b["D"].T @ W_).max() < 1e-13 * N * N
    # boundary interpolation rows are Kronecker deltas for GL
    assert np.array_equal(b["lm1"], np.eye(N + 1)[0]) and np.array_equal(b["lp1"], np.eye(N + 1)[N])


@pytest.mark.parametrize("Nf,Nt", [(1, 1), (3, 3), (6, 2), (2, 6), (8, 5), (4, 8), (7, 1)])
def test_q2_interpolation(orc, Nf, Nt):
    T = orc.interp_matrix(Nf, Nt)
    xf = orc.basis(Nf)["x"]
    xt = orc.basis(Nt)["x"]
    if Nf == Nt:
        assert np.abs(T - np.eye(Nf + 1)).max() < 1e-15
    assert np.abs(T.sum(1) - 1).max() < 1e-14  # partition of unity
    for k in range(0, min(Nf, Nt) + 1):  # reproduces degree <= min(Nf, Nt) exactly
        assert np.abs(T @ xf ** k - xt ** k).max() < 1e-13
    if Nt >= Nf:  # round trip through a richer space is the identity
        T2 = orc.interp_matrix(Nt, Nf)
        assert np.abs(T2 @ T - np.eye(Nf + 1)).max() < 1e-13


@pytest.mark.parametrize("M", range(1, 9))
def test_q2_mortar_projection(orc, M):
    """A6: P^{M->s} is the exact L2 projection: P T = I, conservative."""
    wm = orc.basis(M)["w"]
    for s in range(1, M + 1):
        P = orc.projection_matrix(M, s)
        T = orc.interp_matrix(s, M)
        ws = orc.basis(s)["w"]
        assert np.abs(P @ T - np.eye(s + 1)).max() < 5e-14
        g = np.random.default_rng(M * 10 + s).standard_normal(M + 1)
        assert abs(ws @ (P @ g) - wm @ g) < 1e-13  # conservation of the face integral
        assert np.abs(P @ np.ones(M + 1) - 1).max() < 1e-14


# ----------------------------------------------------------------------------
# Q3 Euler flux and Roe flux
# ----------------------------------------------------------------------------

def test_q3_euler_flux_hand_values(orc):
    q = W.conserved(np.array(1.0), np.array(1.0), np.array(0.0), np.array(0.0), np.array(1.0))
    assert abs(q[4] - 3.0) < 1e-15  # E = p/(g-1) + rho u^2/2 = 2.5 + 0.5
    assert np.abs(orc.euler_flux(q, 0) - [1, 2, 0, 0, 4]).max() < 1e-15
    assert np.abs(orc.euler_flux(q, 1) - [0, 0, 1, 0, 0]).max() < 1e-15
    q0 = W.conserved(np.array(1.0), np.array(0.0), np.array(0.0), np.array(0.0), np.array(1.0))
    for k in range(3):
        ref = np.zeros(5); ref[1 + k] = 1.0
        assert np.abs(orc.euler_flux(q0, k) - ref).max() < 1e-15


def _rand_state(rng, mach=0.5):
    rho = rng.uniform(0.5, 2.0)
    p = rng.uniform(0.5, 2.0)
    c = math.sqrt(1.4 * p / rho)
    u = rng.standard_normal(3) * mach * c / math.sqrt(3)
    return W.conserved(np.array(rho), *[np.array(x) for x in u], np.array(p))


def _unit(rng):
    n = rng.standard_normal(3)
    return n / np.linalg.norm(n)


@pytest.mark.parametrize("flux", ["roe", "llf"])
def test_q3_riemann_consistency_and_symmetry(orc, flux):
    F = orc.roe_flux if flux == "roe" else orc.llf_flux
    rng = np.random.default_rng(1)
    for _ in range(50):
        q, qR, n = _rand_state(rng), _rand_state(rng), _unit(rng)
        fn = sum(n[k] * orc.euler_flux(q, k) for k in range(3))
        assert np.abs(F(q, q, n) - fn).max() < 1e-13 * (1 + np.abs(fn).max())
        # conservation: F(qL, qR, n) = -F(qR, qL, -n)
        assert np.abs(F(q, qR, n) + F(qR, q, -n)).max() < 1e-13 * (1 + np.abs(fn).max())


def test_q3_roe_supersonic_upwinding(orc):
    """All Roe eigenvalues of one sign => F = f(upwind state).n exactly; this
    holds only with Roe's averages (U-property), so it pins the averages and
    the eigen-decomposition."""
    rng = np.random.default_rng(2)
    for sgn in (1.0, -1.0):
        for _ in range(20):
            n = _unit(rng)
            qs = []
            for _ in range(2):
                rho = rng.uniform(0.5, 2.0); p = rng.uniform(0.5, 2.0)
                c = math.sqrt(1.4 * p / rho)
                u = sgn * n * c * rng.uniform(2.5, 4.0) + 0.1 * rng.standard_normal(3)
                qs.append(W.conserved(np.array(rho), *[np.array(x) for x in u], np.array(p)))
            up = qs[0] if sgn > 0 else qs[1]
            ref = sum(n[k] * orc.euler_flux(up, k) for k in range(3))
            got = orc.roe_flux(qs[0], qs[1], n)
            assert np.abs(got - ref).max() < 1e-12 * np.abs(ref).max()


def test_q3_roe_contact_exact(orc):
    """A stationary contact (u_n = 0, equal p, jump in rho) is resolved
    exactly by Roe: mass flux 0, momentum flux = p n."""
    n = np.array([0.0, 1.0, 0.0])
    qL = W.conserved(np.array(1.0), np.array(0.3), np.array(0.0), np.array(0.2), np.array(1.0))
    qR = W.conserved(np.array(2.0), np.array(0.3), np.array(0.0), np.array(0.2), np.array(1.0))
    F = orc.roe_flux(qL, qR, n)
    assert abs(F[0]) < 1e-15 and abs(F[2] - 1.0) < 1e-14 and abs(F[1]) < 1e-15 and abs(F[4]) < 1e-15


def test_q3_viscous_flux_hand_values(orc):
    mu, Pr, g = 0.01, 0.72, 1.4
    ph = orc.phys(orc.NS, mu=mu, Pr=Pr)
    q = W.conserved(np.array(1.0), np.array(0.0), np.array(0.0), np.array(0.0), np.array(1.0))
    alpha = 3.0
    G = np.zeros((3, 5)); G[1, 1] = alpha  # d(rho u)/dy = alpha  => du/dy = alpha
    f = orc.viscous_flux(q, G, 1, ph)  # y flux: tau_xy = mu alpha
    assert np.abs(f - [0, mu * alpha, 0, 0, 0]).max() < 1e-16
    f = orc.viscous_flux(q, G, 0, ph)  # x flux: tau_yx = mu alpha
    assert np.abs(f - [0, 0, mu * alpha, 0, 0]).max() < 1e-16
    G = np.zeros((3, 5)); G[0, 4] = 2.0  # dE/dx = 2 at rest => dp/dx = 0.8, dT/dx = 0.8
    kappa = mu * g / ((g - 1) * Pr)
    f = orc.viscous_flux(q, G, 0, ph)
    assert np.abs(f - [0, 0, 0, 0, kappa * 0.8]).max() < 1e-15
    G = np.zeros((3, 5)); G[0, 1] = 1.0  # du/dx = 1: tau_xx = 4/3 mu, tau_yy = -2/3 mu
    assert abs(orc.viscous_flux(q, G, 0, ph)[1] - 4.0 / 3.0 * mu) < 1e-16
    assert abs(orc.viscous_flux(q, G, 1, ph)[2] + 2.0 / 3.0 * mu) < 1e-16


# ----------------------------------------------------------------------------
# Q4 free-stream preservation, Q6 conservation
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("layout", ["uniform3", "uniform8", "mixed"])
def test_q4_freestream_cube(orc, layout):
    m = W.cube_mesh(4)
    P = orc.Problem(m)
    o = {"uniform3": W.orders_uniform(m.E, 3), "uniform8": W.orders_uniform(m.E, 8),
         "mixed": W.orders_random(m.E, 1, 8, 3)}[layout]
    q = W.uniform_state(o)
    for var in (orc.NONISOLATED, orc.ISOLATED):
        assert np.abs(P.rhs(o, q, var)).max() < 1e-11  # |f| ~ 4, (N+1)^2/h ~ 300


@pytest.mark.parametrize("physics", ["euler", "ns"])
def test_q4_freestream_ogrid(orc, physics):
    # Free stream is preserved on curved p-nonconforming faces when both sides
    # resolve the face metric polynomial: Ja^1 has degree g-1 in eta, Ja^3 =
    # (0, 0, x_xi y_eta - x_eta y_xi) has degree 2g-1 in eta (DESIGN.md,
    # "Free-stream condition").  g = 2 here, so N_eta >= 3.
    m = W.ogrid_mesh(4, 8, 2, g_eta=2)
    m.nbr[m.nbr == W.BC_WALL] = W.BC_FARFIELD  # free stream everywhere
    nsp = W.ns_params()
    ph = orc.phys(orc.NS if physics == "ns" else orc.EULER, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
    P = orc.Problem(m, ph)
    o = W.orders_random(m.E, (1, 3, 1), (8, 8, 3), 7)
    q = W.uniform_state(o, vel=(1.0, 0.0, 0.0), p=nsp["p_inf"])
    scale = np.abs(nsp["qinf"]).max()
    for var in (orc.NONISOLATED, orc.ISOLATED):
        assert np.abs(P.rhs(o, q, var)).max() < 1e-12 * scale * 100


def test_q4_rest_state_with_walls(orc):
    m = W.ogrid_mesh(4, 8, 1, g_eta=4)
    nsp = W.ns_params()
    rest = W.conserved(np.array(1.0), np.array(0.0), np.array(0.0), np.array(0.0), np.array(nsp["p_inf"]))
    P = orc.Problem(m, orc.phys(orc.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=rest))
    o = W.orders_random(m.E, (4, 4, 1), (6, 6, 2), 8)
    q = W.uniform_state(o, vel=(0, 0, 0), p=nsp["p_inf"])
    assert np.abs(P.rhs(o, q)).max() < 1e-9  # p_inf ~ 17.9


def _sum_M_qdot(P, o, r):
    M = P.mass(o)
    offm = W.offsets(o, 1)
    tot = np.zeros(5); ab = np.zeros(5)
    for e, blk in _blocks(r, o):
        w = M[offm[e]:offm[e + 1]]
        tot += (blk * w).sum(1)
        ab += np.abs(blk * w).sum(1)
    return tot, ab


@pytest.mark.parametrize("layout,physics", [("uniform", "euler"), ("mixed", "euler"), ("mixed", "ns")])
def test_q6_conservation(orc, layout, physics):
    m = W.cube_mesh(4)
    ph = orc.phys(orc.NS if physics == "ns" else orc.EULER, mu=0.01, Pr=0.72)
    P = orc.Problem(m, ph)
    o = W.orders_uniform(m.E, 4) if layout == "uniform" else W.orders_random(m.E, 1, 7, 11)
    X = P.node_coords(o)
    q = W.pulse_state(X, o, center=(0.3, 0.6, 0.5), sigma=0.12)
    r = P.rhs(o, q)
    tot, ab = _sum_M_qdot(P, o, r)
    assert np.all(np.abs(tot) < 1e-13 * ab)
    # the isolated operator is NOT conservative for discontinuous data
    ri = P.rhs(o, q, orc.ISOLATED)
    toti, abi = _sum_M_qdot(P, o, ri)
    if layout == "mixed":
        assert np.abs(toti[0]) > 1e-8 * abi[0]


# ----------------------------------------------------------------------------
# Q5 exact differentiation of polynomials
# ----------------------------------------------------------------------------

def test_q5_exact_polynomial(orc):
    """rho a polynomial of degree <= N_d per direction, u, p constant =>
    Qdot = -(u.grad rho)(1, u, |u|^2/2) exactly at the nodes (flux affine in
    rho).  Isolated everywhere; non-isolated on elements away from the
    periodic wrap (data continuous across their faces)."""
    m = W.cube_mesh(4)
    P = orc.Problem(m)
    o = W.orders_random(m.E, 2, 6, 5)
    o[:] = np.maximum(o, 2)
    X = P.node_coords(o)
    vel = np.array([1.0, 0.5, 0.25])
    q = np.empty(P.size(o)); ref = np.empty_like(q)
    offx = W.offsets(o, 3); offq = W.offsets(o, 5)
    for e in range(m.E):
        n = (offx[e + 1] - offx[e]) // 3
        x, y, z = X[offx[e]:offx[e + 1]].reshape(3, n)
        rho = 1.0 + 0.2 * x - 0.1 * y * y + 0.05 * x * z  # degree <= 2 per direction
        gr = np.stack([0.2 + 0.05 * z, -0.2 * y, 0.05 * x])
        q[offq[e]:offq[e + 1]] = W.conserved(rho, *(vel[k] * np.ones(n) for k in range(3)), np.ones(n)).ravel()
        ug = vel @ gr
        ref[offq[e]:offq[e + 1]] = (-ug * np.stack([np.ones(n), vel[0] * np.ones(n), vel[1] * np.ones(n),
                                                   vel[2] * np.ones(n), 0.5 * vel @ vel * np.ones(n)])).ravel()
    ri = P.rhs(o, q, orc.ISOLATED)
    assert np.abs(ri - ref).max() < 1e-11
    rn = P.rhs(o, q)
    for e in range(m.E):
        i, j, k = e % 4, (e // 4) % 4, e // 16
        if 0 < i < 3 and 0 < j < 3 and 0 < k < 3:
            assert np.abs(rn[offq[e]:offq[e + 1]] - ref[offq[e]:offq[e + 1]]).max() < 1e-11


def test_q5_br1_gradient_exact(orc):
    """BR1 gradient of a field of degree <= N per element is exact (affine),
    isolated; and a constant field has zero gradient on the curved O-grid."""
    m = W.cube_mesh(2)
    P = orc.Problem(m, orc.phys(orc.NS, mu=0.01))
    o = W.orders_uniform(m.E, 3)
    X = P.node_coords(o)
    offx = W.offsets(o, 3); offq = W.offsets(o, 5); offg = W.offsets(o, 15)
    q = np.empty(P.size(o)); ref = np.empty(P.size(o, 15))
    for e in range(m.E):
        n = (offx[e + 1] - offx[e]) // 3
        x, y, z = X[offx[e]:offx[e + 1]].reshape(3, n)
        f = np.stack([1 + x * y, 2 + z ** 3, x ** 2, y * z * x, 3 + y])
        gx = np.stack([y, 0 * x, 2 * x, y * z, 0 * x])
        gy = np.stack([x, 0 * x, 0 * x, x * z, 1 + 0 * x])
        gz = np.stack([0 * x, 3 * z ** 2, 0 * x, x * y, 0 * x])
        q[offq[e]:offq[e + 1]] = f.ravel()
        ref[offg[e]:offg[e + 1]] = np.concatenate([gx.ravel(), gy.ravel(), gz.ravel()])
    g = P.gradient(o, q, orc.ISOLATED)
    assert np.abs(g - ref).max() < 1e-12
    mo = W.ogrid_mesh(3, 8, 1, g_eta=4)
    Po = orc.Problem(mo, orc.phys(orc.NS, mu=0.01, qinf=W.conserved(*[np.array(v) for v in (1.0, 0, 0, 0, 1.0)])))
    oo = W.orders_uniform(mo.E, 4)
    qc = W.uniform_state(oo, vel=(0, 0, 0), p=1.0)
    assert np.abs(Po.gradient(oo, qc)).max() < 1e-11


# ----------------------------------------------------------------------------
# Q7 / Q8 / Q10 tau-estimation
# ----------------------------------------------------------------------------

def _pulse_problem(orc, n=4, N=6, sigma=0.1, center=(0.5, 0.5, 0.5)):
    m = W.cube_mesh(n)
    P = orc.Problem(m)
    o = W.orders_uniform(m.E, N)
    X = P.node_coords(o)
    q = W.pulse_state(X, o, center=center, sigma=sigma)
    return m, P, o, X, q


def test_q8_tau_zero_at_fine_order_and_traditional_scaling(orc):
    m, P, o, X, q = _pulse_problem(orc, n=2, N=5)
    r = P.rhs(o, q, orc.ISOLATED)  # SAME reference (A4)
    for d in range(3):
        t = P.tau_field(o, q, r, e=3, d=d, p=5)  # p = N: I is the identity
        assert np.abs(t).max() == 0.0
    # tau_trad = J w w w tau_new nodewise
    e, d, p = 5, 1, 3
    tn = P.tau_field(o, q, r, e, d, p, orc.TAU_NEW)
    tt = P.tau_field(o, q, r, e, d, p, orc.TAU_TRADITIONAL)
    O = [5, 5, 5]; O[d] = p
    J = m.extra["h"][0] ** 3 / 8
    wx, wy, wz = (orc.basis(O[k])["w"] for k in range(3))
    Mw = J * (wz[:, None, None] * wy[None, :, None] * wx[None, None, :]).ravel()
    assert np.abs(tt - tn * Mw).max() < 1e-13 * np.abs(tt).max()


def test_q8_tau_directional_structure(orc):
    """x-only field => tau_y = tau_z = 0 (roundoff); swapping x and y in the
    data swaps tau_x and tau_y."""
    m = W.cube_mesh(3)
    P = orc.Problem(m)
    o = W.orders_uniform(m.E, 5)
    X = P.node_coords(o)
    offx = W.offsets(o, 3)

    def state(fn, vel):
        q = np.empty(P.size(o))
        offq = W.offsets(o, 5)
        for e in range(m.E):
            n = (offx[e + 1] - offx[e]) // 3
            x, y, z = X[offx[e]:offx[e + 1]].reshape(3, n)
            rho = fn(x, y, z)
            q[offq[e]:offq[e + 1]] = W.conserved(rho, *(vel[k] * np.ones(n) for k in range(3)), np.ones(n)).ravel()
        return q

    q = state(lambda x, y, z: 1 + 0.1 * np.sin(2 * np.pi * x), (1.0, 0.5, 0.25))
    tau = P.tau_estimate(o, q, P.rhs(o, q, orc.ISOLATED))
    assert tau[:, 0, 1:5].max() > 1e-4
    assert tau[:, 1:, 1:5].max() < 1e-12 * tau[:, 0, 1:5].max() * 1e3
    f = lambda x, y, z: 1 + 0.1 * np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y) + 0.05 * np.sin(2 * np.pi * z)
    qa = state(f, (1.0, 0.5, 0.25))
    qb = state(lambda x, y, z: f(y, x, z), (0.5, 1.0, 0.25))
    ta = P.tau_estimate(o, qa, P.rhs(o, qa, orc.ISOLATED))
    tb = P.tau_estimate(o, qb, P.rhs(o, qb, orc.ISOLATED))
    perm = np.array([(e % 3) * 3 + (e // 3) % 3 + 9 * (e // 9) for e in range(m.E)])  # (i,j,k)->(j,i,k)
    perm = np.array([((e // 3) % 3) + 3 * (e % 3) + 9 * (e // 9) for e in range(m.E)])
    assert np.allclose(tb[perm][:, 1, 1:5], ta[:, 0, 1:5], rtol=1e-10, atol=1e-12)
    assert np.allclose(tb[perm][:, 0, 1:5], ta[:, 1, 1:5], rtol=1e-10, atol=1e-12)


def test_q7_exact_truncation_error(orc):
    """GTEE with the exact operator: the pulse is an exact Euler
    solution with F(q) = (u.grad rho)(1, u, |u|^2/2).  Feeding -F as the
    reference gives the exact tau~(p); it vanishes when the data are
    polynomials of degree <= p along d, and the SAME-reference estimate
    differs from it by exactly -I_p tau~(N), bounded by the
    interpolation constant times ||tau~(N)||."""
    m = W.cube_mesh(2)
    P = orc.Problem(m)
    o = W.orders_uniform(m.E, 6)
    X = P.node_coords(o)
    offx = W.offsets(o, 3); offq = W.offsets(o, 5)
    vel = np.array([1.0, 0.5, 0.25])
    q = np.empty(P.size(o)); F = np.empty_like(q)
    for e in range(m.E):
        n = (offx[e + 1] - offx[e]) // 3
        x, y, z = X[offx[e]:offx[e + 1]].reshape(3, n)
        rho = 1 + 0.1 * np.exp(-((x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2) / 0.02)
        dr = np.stack([-(x - 0.5), -(y - 0.5), -(z - 0.5)]) / 0.01 * (rho - 1)
        q[offq[e]:offq[e + 1]] = W.conserved(rho, *(vel[k] * np.ones(n) for k in range(3)), np.ones(n)).ravel()
        ug = vel @ dr
        F[offq[e]:offq[e + 1]] = (ug * np.stack([np.ones(n), vel[0] * np.ones(n), vel[1] * np.ones(n),
                                                 vel[2] * np.ones(n), 0.5 * vel @ vel * np.ones(n)])).ravel()
    exact = P.tau_estimate(o, q, -F)
    same = P.tau_estimate(o, q, P.rhs(o, q, orc.ISOLATED))
    tauN = np.abs(-P.rhs(o, q, orc.ISOLATED) - F).max()  # ||tau~(N)||_inf
    for d in range(3):
        for p in range(1, 6):
            assert np.all(np.abs(same[:, d, p] - exact[:, d, p]) <= 2.0 * tauN)
    # polynomial data of degree <= p along x: exact tau~ vanishes for that p
    for e in range(m.E):
        n = (offx[e + 1] - offx[e]) // 3
        x = X[offx[e]:offx[e + 1]].reshape(3, n)[0]
        rho = 1 + 0.1 * x + 0.2 * x * x
        q[offq[e]:offq[e + 1]] = W.conserved(rho, *(vel[k] * np.ones(n) for k in range(3)), np.ones(n)).ravel()
        ug = vel[0] * (0.1 + 0.4 * x)
        F[offq[e]:offq[e + 1]] = (ug * np.stack([np.ones(n), vel[0] * np.ones(n), vel[1] * np.ones(n),
                                                 vel[2] * np.ones(n), 0.5 * vel @ vel * np.ones(n)])).ravel()
    ex = P.tau_estimate(o, q, -F)
    assert ex[:, 0, 2:6].max() < 1e-12 and ex[:, 0, 1].min() > 1e-3


def test_q10_spectral_decay_cfg2_setting(orc):
    """tau decays exponentially for smooth solutions.  cfg2 setting
    (h = 1/16, sigma = 0.08, N = 6), SAME reference, elements carrying the
    pulse: tau_d(p) strictly decreasing, fitted slope < 0."""
    m = W.cube_mesh(16)
    # restrict to a 6x6x6 block of elements around the centre for speed
    P = orc.Problem(m)
    o = W.orders_uniform(m.E, 6)
    X = P.node_coords(o)
    q = W.pulse_state(X, o, center=(0.5, 0.5, 0.5), sigma=0.08)
    r = P.rhs(o, q, orc.ISOLATED)
    tau = P.tau_estimate(o, q, r)
    sup = tau[:, 0, 0] > 1e-3 * tau[:, 0, 0].max()
    assert sup.sum() > 100
    t = tau[sup][:, :, 1:6]
    assert np.all(np.diff(t, axis=2) < 0)
    _, slopes = orc.build_map(o[sup], tau[sup], 3, 8)
    assert np.all(slopes < 0)


# ----------------------------------------------------------------------------
# Q11 RK3, Q12 dt
# ----------------------------------------------------------------------------

def test_q12_dt_closed_form(orc):
    m = W.cube_mesh(4)
    P = orc.Problem(m)
    for N in (3, 6):
        o = W.orders_uniform(m.E, N)
        q = W.uniform_state(o, vel=(1.0, 0.5, 0.25), p=1.0)
        c = math.sqrt(1.4)
        ref = 0.5 * 0.25 / (sum(abs(u) + c for u in (1.0, 0.5, 0.25)) * (N + 1) ** 2)
        assert abs(P.dt(o, q, 0.5) - ref) <= 1e-15 * ref  # a few ulp


def test_q11_rk3_constant_state_and_order(orc):
    m = W.cube_mesh(2)
    P = orc.Problem(m)
    o = W.orders_uniform(m.E, 2)
    qc = W.uniform_state(o)
    assert np.array_equal(P.rk3_step(o, qc, 1e-3), qc)  # N=2: Qdot == 0 exactly
    o = W.orders_uniform(m.E, 5)
    X = P.node_coords(o)
    q0 = W.pulse_state(X, o, sigma=0.15)
    T = 0.02

    def run(k):
        q = q0
        for _ in range(k):
            q = P.rk3_step(o, q, T / k)
        return q

    ref = run(64)
    errs = [np.abs(run(k) - ref).max() for k in (2, 4, 8)]
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert all(2.8 < r < 3.3 for r in orders), orders


# ----------------------------------------------------------------------------
# Q13-Q15 extrapolation, selection, Table 1, jump fixpoint; Q16 transfer
# ----------------------------------------------------------------------------

def test_q13_extrapolation(orc):
    E = 1
    o = np.array([[5, 4, 2]], np.int32)
    tau = np.full((E, 3, 9), np.nan)
    tau[0, :, 0] = 1.0
    tau[0, 0, 1:5] = 10.0 ** -np.arange(1, 5)  # exact exponential: a = 0, b = -1
    tau[0, 1, 1:4] = [1e-2, 2e-2, 5e-3]        # non-monotone, slope > 0? fit decides
    tau[0, 2, 1] = 1e-3                        # N = 2: a single point, no extrapolation
    mp, sl = orc.build_map(o, tau, 1, 8)
    assert abs(sl[0, 0] + 1.0) < 1e-12
    # hat_x(n) = 10^-n for all n; y, z at n = 1 are the measured values
    for n1 in range(1, 9):
        assert abs(mp[0, 0, 0, n1 - 1] - (10.0 ** -n1 + 1e-2 + 1e-3)) < 1e-12 * (10.0 ** -n1 + 1.1e-2)
    assert mp[0, 0, 0, 0] < 1.0
    # z at N_z = 2: no extrapolation possible, the order is kept (P:592,
    # reading R12): hat_z(2) = 0, hat_z(n > 2) = sentinel
    assert abs(mp[0, 1, 0, 0] - (0.1 + 1e-2)) < 1e-14
    assert mp[0, 2, 0, 0] >= 1e30
    # y: log10 fit over (1e-2, 2e-2, 5e-3): slope = (log10(5e-3) - log10(1e-2)) / 2 < 0 => asymptotic
    b = (math.log10(5e-3) - math.log10(1e-2)) / 2
    a = np.mean(np.log10([1e-2, 2e-2, 5e-3])) - 2 * b
    assert abs(sl[0, 1] - b) < 1e-12
    assert abs(mp[0, 0, 5, 0] - (0.1 + 10 ** (a + 6 * b) + 1e-3)) < 1e-12
    # resolved direction (max tau <= 1e-13 max(1, |R|)) => hat == 0 everywhere
    tau2 = tau.copy(); tau2[0, 0, 1:5] = 1e-15
    mp2, _ = orc.build_map(o, tau2, 1, 8)
    assert mp2[0, 0, 0, 7] == mp2[0, 0, 0, 0]
    # R11: a direction at rounding level next to the element's others (here z,
    # 1e-12 against x's 1e-1: above the A14 floor, growing with p, so
    # non-asymptotic) is resolved, not a sentinel; at 1e-7 of the others it
    # is estimated (sentinel for n_z >= N_z)
    o4 = np.array([[5, 5, 5]], np.int32)
    tau4 = np.full((1, 3, 9), np.nan)
    tau4[0, :, 0] = 1e-3
    tau4[0, 0, 1:5] = [1e-1, 1e-2, 1e-3, 1e-4]
    tau4[0, 1, 1:5] = [1e-2, 1e-3, 1e-4, 1e-5]
    tau4[0, 2, 1:5] = [1e-12, 2e-12, 3e-12, 4e-12]
    mp4, _ = orc.build_map(o4, tau4, 5, 8)
    assert np.all(mp4 < 1e30) and np.all(mp4[1:] == mp4[0])  # independent of n_z
    tau4[0, 2, 1:5] = [1e-8, 2e-8, 3e-8, 4e-8]
    mp5, _ = orc.build_map(o4, tau4, 5, 8)
    assert np.all(mp5 >= 1e30)
    # N_d = 1: keep the order
    o3 = np.array([[1, 4, 2]], np.int32)
    mp3, _ = orc.build_map(o3, tau, 1, 8)
    assert mp3[0, 0, 0, 0] < 1 and mp3[0, 0, 0, 1] >= 1e30


def test_q14_selection_brute_force(orc):
    rng = np.random.default_rng(14)
    Nmin, Nmax = 2, 6
    K = Nmax - Nmin + 1
    mp = 10.0 ** rng.uniform(-6, 0, size=(1000, K, K, K))
    tau_max = 1e-3
    sel, mg = orc.select_from_map(mp, Nmin, Nmax, tau_max)
    for e in range(1000):
        best = None
        for n1 in range(Nmin, Nmax + 1):
            for n2 in range(Nmin, Nmax + 1):
                for n3 in range(Nmin, Nmax + 1):
                    if mp[e, n3 - Nmin, n2 - Nmin, n1 - Nmin] < tau_max:
                        key = ((n1 + 1) * (n2 + 1) * (n3 + 1), n1 + n2 + n3, (n1, n2, n3))
                        best = key if best is None or key < best else best
        exp = best[2] if best else (Nmax,) * 3
        assert tuple(sel[e]) == exp


def test_q14_table1(orc):
    g = json.load(open(os.path.join(GOLD, "table1.json")))
    Nmin, Nmax, tmax = g["Nmin"], g["Nmax"], 1.0
    K = Nmax - Nmin + 1

    def stage_map(feas):
        mp = np.full((1, K, K, K), 2 * tmax)  # [e, n3, n2, n1]; n3 pinned to N_min (2-D element)
        for n1, n2 in feas:
            mp[0, 0, n2 - Nmin, n1 - Nmin] = tmax / 2
        return mp

    maps = [stage_map(f) for f in g["stage_feasible"]]
    # approach 1 + F_max: select per stage, then max
    picks = [tuple(orc.select_from_map(mp, Nmin, Nmax, tmax)[0][0][:2]) for mp in maps]
    assert [list(p) for p in picks] == g["stage_selected_approach1"]
    a1 = tuple(max(p[i] for p in picks) for i in range(2))
    assert list(a1) == g["approach1_Fmax"] and (a1[0] + 1) * (a1[1] + 1) == g["approach1_NDOF"]
    # approach 2 (eq totalTruncMap) + F_max: combine maps, select once
    total = np.zeros_like(maps[0])
    for mp in maps:
        total = orc.combine_max(total, mp)
    a2 = tuple(orc.select_from_map(total, Nmin, Nmax, tmax)[0][0][:2])
    assert list(a2) == g["approach2_Fmax"] and (a2[0] + 1) * (a2[1] + 1) == g["approach2_NDOF"]


def test_q14_table1_f_av(orc):
    """F_av on Table 1: approach 1 averages the
    stage picks (1,3) and (3,1) to (2,2) -- by hand, NDOF 9 -- and approach 2
    with the averaged map keeps exactly the combinations feasible in both
    stages (tau_max/2 stays feasible, (tau_max/2 + 2 tau_max)/2 does not) ->
    (2,2).  Half-up rounding (reading R8): picks 2 and 3 average to 3."""
    g = json.load(open(os.path.join(GOLD, "table1.json")))
    Nmin, Nmax, tmax = g["Nmin"], g["Nmax"], 1.0
    K = Nmax - Nmin + 1

    def stage_map(feas):
        mp = np.full((1, K, K, K), 2 * tmax)
        for n1, n2 in feas:
            mp[0, 0, n2 - Nmin, n1 - Nmin] = tmax / 2
        return mp

    maps = [stage_map(f) for f in g["stage_feasible"]]
    picks = [orc.select_from_map(mp, Nmin, Nmax, tmax)[0] for mp in maps]
    assert list(orc.combine_degrees(picks, 1)[0][:2]) == [2, 2]
    assert list(orc.combine_degrees(picks, 0)[0][:2]) == g["approach1_Fmax"]
    total = np.zeros_like(maps[0])
    for mp in maps:
        total = orc.combine_sum(total, mp)
    assert list(orc.select_from_map(total / len(maps), Nmin, Nmax, tmax)[0][0][:2]) == [2, 2]
    assert orc.combine_degrees([[[2, 2, 2]], [[3, 2, 1]]], 1).tolist() == [[3, 2, 2]]


def test_q15_jump_cones(orc):
    m = W.cube_mesh(15, 1, 1)
    o = np.ones((15, 3), np.int32)
    o[7, 0] = 8
    ob, _ = orc.jump_fixpoint(m.nbr, o, orc.JUMP_B, 8)
    assert list(ob[:, 0]) == [1, 2, 3, 4, 5, 6, 7, 8, 7, 6, 5, 4, 3, 2, 1]
    oa, _ = orc.jump_fixpoint(m.nbr, o, orc.JUMP_A, 8)
    assert list(oa[:, 0]) == [1, 1, 1, 1, 2, 3, 5, 8, 5, 3, 2, 1, 1, 1, 1]
    assert np.all(ob[:, 1:] == 1) and np.all(oa[:, 1:] == 1)


def test_q15_jump_least_fixpoint_brute(orc):
    rng = np.random.default_rng(15)
    for trial in range(6):
        m = W.cube_mesh(4, 3, 2)
        o = rng.integers(1, 9, size=(m.E, 3)).astype(np.int32)
        for rule in (orc.JUMP_A, orc.JUMP_B):
            out, _ = orc.jump_fixpoint(m.nbr, o, rule, 8)
            r = (lambda x: (2 * x) // 3) if rule == orc.JUMP_A else (lambda x: x - 1)
            # satisfies the rule on every face, never lowers
            assert np.all(out >= o)
            for e in range(m.E):
                for f in range(6):
                    assert np.all(out[e] >= np.minimum(8, r(out[m.nbr[e, f]])))
            # least: Gauss-Seidel brute force from the input reaches the same point
            gs = o.copy()
            changed = True
            while changed:
                changed = False
                for e in range(m.E):
                    for d in range(3):
                        v = max([gs[e, d]] + [r(gs[m.nbr[e, f], d]) for f in range(6)])
                        v = min(8, v)
                        if v != gs[e, d]:
                            gs[e, d] = v
                            changed = True
            assert np.array_equal(gs, out)
        oa, _ = orc.jump_fixpoint(m.nbr, o, orc.JUMP_A, 8)
        ob, _ = orc.jump_fixpoint(m.nbr, o, orc.JUMP_B, 8)
        assert W.ndof(ob) >= W.ndof(oa)


def test_q16_transfer(orc):
    m = W.cube_mesh(2)
    P = orc.Problem(m)
    o = W.orders_random(m.E, 2, 5, 16)
    X = P.node_coords(o)
    q = W.pulse_state(X, o, sigma=0.2)
    hi = np.minimum(o + 3, 8).astype(np.int32)
    up = orc.transfer(o, q, hi)
    back = orc.transfer(hi, up, o)
    assert np.abs(back - q).max() < 1e-13
    # element means preserved on raise (quadrature exact for the interpolant)
    Mo, Mh = P.mass(o), P.mass(hi)
    offo, offh = W.offsets(o, 1), W.offsets(hi, 1)
    for (e, bo), (_, bh) in zip(_blocks(q, o), _blocks(up, hi)):
        mo = (bo * Mo[offo[e]:offo[e + 1]]).sum(1) / Mo[offo[e]:offo[e + 1]].sum()
        mh = (bh * Mh[offh[e]:offh[e + 1]]).sum(1) / Mh[offh[e]:offh[e + 1]].sum()
        assert np.abs(mo - mh).max() < 1e-13
    qc = W.uniform_state(o)
    assert np.abs(orc.transfer(o, qc, hi) - W.uniform_state(hi)).max() < 1e-13


# ----------------------------------------------------------------------------
# Q17 non-isolated tau-estimation (reading R7)
# ----------------------------------------------------------------------------

def _entropy_wave(X, orders, slope=0.1, gamma=1.4):
    """rho = 1 + slope*x, u = (1,0,0), p = 1: the Euler flux is linear in q
    (f = u q + p e_x-terms with u, p constant), so every DGSEM operator is
    exact on it wherever the state is continuous; the periodic wrap x=1|0
    carries the only jump."""
    off3, off5 = W.offsets(orders, 3), W.offsets(orders, 5)
    q = np.empty(off5[-1])
    for e in range(len(orders)):
        n = (off3[e + 1] - off3[e]) // 3
        x = X[off3[e]:off3[e] + n]
        rho = 1.0 + slope * x
        b = q[off5[e]:off5[e + 1]].reshape(5, n)
        b[0] = rho
        b[1] = rho
        b[2] = 0.0
        b[3] = 0.0
        b[4] = 1.0 / (gamma - 1.0) + 0.5 * rho
    return q


def test_q17_noniso_tau_freestream(orc):
    m = W.cube_mesh(3, 2, 2)
    P = orc.Problem(m)
    o = W.orders_random(m.E, 2, 6, 17)
    q = W.uniform_state(o)
    R = P.rhs(o, q)
    for form in (orc.TAU_NEW, orc.TAU_TRADITIONAL):
        t = P.tau_estimate_noniso(o, q, R, form)
        lv = t[:, :, 1:]
        assert np.nanmax(np.abs(lv)) < 1e-11
        # defined exactly for p < N_d (reading R1), slot 0 = ||R||_inf
        for e in range(m.E):
            for d in range(3):
                assert np.all(np.isfinite(t[e, d, 1:o[e, d]])) and np.all(np.isnan(t[e, d, o[e, d]:]))


def test_q17_noniso_tau_jump_pattern(orc):
    """Entropy wave with one jump (periodic wrap in x, u = +1): the Roe flux of
    a pure entropy jump is the upwind flux F(q_L) (wave strengths a1 = a5 = 0),
    so only the downwind element (ix = 0) sees the jump in its lifting.  The
    non-isolated tau is zero (to rounding) except for direction x at that
    element; the isolated tau (element-local coarse residual, same SOLVER
    reference) is nonzero there for EVERY direction (it misses the jump's
    lifting) -- a dropped face term, a wrong sign, swapped face sides, a
    misaligned neighbour trace or a transposed interpolation breaks one of
    these."""
    nx = 4
    m = W.cube_mesh(nx, 2, 2)
    P = orc.Problem(m)
    o = W.orders_uniform(m.E, 4)
    q = _entropy_wave(P.node_coords(o), o)
    R = P.rhs(o, q)
    scale = np.abs(R).max()
    tn = P.tau_estimate_noniso(o, q, R)
    ti = P.tau_estimate(o, q, R)
    ix = np.arange(m.E) % nx
    wrap = ix == 0  # downwind of the jump
    for d in range(3):
        lv_n, lv_i = tn[:, d, 1:4], ti[:, d, 1:4]
        assert np.all(lv_i[~wrap] < 1e-10 * scale)
        assert np.all(lv_i[wrap] > 1e-3 * scale)
        assert np.all(lv_n[~wrap] < 1e-10 * scale)
        if d == 0:
            assert np.all(lv_n[wrap] > 1e-3 * scale)
        else:
            assert np.all(lv_n[wrap] < 1e-10 * scale)


# ----------------------------------------------------------------------------
# Q18 L2-projection restriction for the tau-estimate (the A3 flag, SURVEY 8(f)
# rank 4): P^{N->p} along one direction
# ----------------------------------------------------------------------------

def test_q18_restrict_l2_line_integrals(orc):
    """Along the restricted direction every line keeps its integral (P^{N->p}
    is the L2 projection onto degree p, which contains the constants; GL with
    p+1 / N+1 points integrates degree p / N exactly), and data of degree <= p
    along that direction is reproduced exactly (= interpolation)."""
    m = W.cube_mesh(1)
    P = orc.Problem(m)
    o = np.array([[4, 5, 6]], np.int32)
    rng = np.random.default_rng(18)
    q = rng.standard_normal(P.size(o))
    X = P.node_coords(o)
    for d in range(3):
        for p in range(1, int(o[0, d])):
            oc = o.copy()
            oc[0, d] = p
            qc = orc.restrict_l2(o, q, oc, d)
            # whole-element weighted sums (J w w w), affine element: line integrals summed
            M, Mc = P.mass(o), P.mass(oc)
            a = q.reshape(5, -1) @ M
            b = qc.reshape(5, -1) @ Mc
            assert np.abs(a - b).max() < 1e-13 * np.abs(q).max()
            # a state linear in x_d is reproduced: projection == interpolation
            lin = np.tile(1.0 + 0.3 * X[d * X.size // 3:(d + 1) * X.size // 3], 5)
            assert np.abs(orc.restrict_l2(o, lin, oc, d) - orc.transfer(o, lin, oc)).max() < 1e-14


def test_q18_tau_projection_vs_interpolation(orc):
    """On the entropy wave of Q17 (linear in x, constant in y, z) the two
    restrictions agree wherever the restricted data is a polynomial of degree
    <= p along d (away from the jump's lifting), and they differ on a pulse."""
    nx = 4
    m = W.cube_mesh(nx, 2, 2)
    P = orc.Problem(m)
    o = W.orders_uniform(m.E, 4)
    q = _entropy_wave(P.node_coords(o), o)
    R = P.rhs(o, q)
    ti, tp = P.tau_estimate(o, q, R), P.tau_estimate(o, q, R, restriction=1)
    ni, np_ = P.tau_estimate_noniso(o, q, R), P.tau_estimate_noniso(o, q, R, restriction=1)
    scale = np.abs(R).max()
    ix = np.arange(m.E) % nx
    for d in range(3):
        sel = ix != 0 if d == 0 else slice(None)
        assert np.abs(ti[sel, d, 1:4] - tp[sel, d, 1:4]).max() < 1e-10 * scale
        assert np.abs(ni[sel, d, 1:4] - np_[sel, d, 1:4]).max() < 1e-10 * scale
    qp = W.pulse_state(P.node_coords(o), o, sigma=0.15)
    Rp = P.rhs(o, qp)
    a, b = P.tau_estimate(o, qp, Rp), P.tau_estimate(o, qp, Rp, restriction=1)
    assert np.nanmax(np.abs(a[:, :, 1:] - b[:, :, 1:])) > 1e-6 * np.nanmax(np.abs(a[:, :, 1:]))
