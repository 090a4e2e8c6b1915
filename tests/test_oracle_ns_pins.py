"""Closed-form pins of the oracle's Navier-Stokes path (CPU, -m "not gpu").

Each pin fixes a part of ``oracle/dgsem_oracle.c`` that the structural pins
(free stream, conservation, rest state) cannot see, against a value the
mathematics fixes independently of the oracle:

* Q19 exact NS solutions of polynomial form (P:106-126 eqs SystemAdvDiff,
  first-order system with g = grad q; P:119-140 eqs DGSEMsystem:1-2, BR1
  P:472).  With GL nodes and data of degree <= N per element the discrete
  operator differentiates exactly, so Qdot equals the analytic time
  derivative at the nodes: the sign and the 1/2 of the viscous terms, the
  2/3 divergence term, kappa = mu gamma / ((gamma-1) Pr) and the BR1 face
  averages (non-isolated, element away from the periodic wrap) are fixed.
* Q20 the viscous step bound (reading A11) in closed form.
* Q21 wall faces (reading A10): the discrete flux balance sum M Qdot =
  -oint F.n dA with the no-slip adiabatic wall flux, in closed form for a
  channel flow (wall shear, wall pressure, zero heat flux).
* Q22 the BR1 gradient obeys the discrete Gauss theorem with the face state
  qhat (summation by parts; P:137-140 eq DGSEMsystem:2).
* Q23 the dynamic decrease cap (A16) properties.
* Q9  decoupling of the directional estimates (reading A12): for an affine
  flux the full tau-field of a simultaneous coarsening equals the sum of the
  directional fields interpolated in the other directions.

tests/test_oracle_mutations.py compiles mutated copies of the oracle (sign /
factor flips) and shows each of these pins fails on them.
"""
import math

import numpy as np
import pytest

import oracle as O
import workloads as W

GAMMA = 1.4


def _fields(X, orders, fn):
    """Conserved state from a primitive-field function fn(x, y, z) ->
    (rho, u, v, w, p) evaluated at the node coordinates."""
    offx = W.offsets(orders, 3)
    offq = W.offsets(orders, 5)
    q = np.empty(offq[-1])
    for e in range(len(orders)):
        n = (offx[e + 1] - offx[e]) // 3
        x, y, z = X[offx[e]:offx[e + 1]].reshape(3, n)
        q[offq[e]:offq[e + 1]] = W.conserved(*fn(x, y, z)).ravel()
    return q


def _expect(X, orders, fn):
    offx = W.offsets(orders, 3)
    offq = W.offsets(orders, 5)
    r = np.empty(offq[-1])
    for e in range(len(orders)):
        n = (offx[e + 1] - offx[e]) // 3
        x, y, z = X[offx[e]:offx[e + 1]].reshape(3, n)
        r[offq[e]:offq[e + 1]] = np.stack([np.broadcast_to(c, x.shape) for c in fn(x, y, z)]).ravel()
    return r


def _channel_mesh(ny, walls=False, L=(0.7, 1.0, 0.6)):
    m = W.cube_mesh(2, ny, 2, L=L)
    if walls:
        for e in range(m.E):
            j = (e // 2) % ny
            if j == 0:
                m.nbr[e, 2] = W.BC_WALL
            if j == ny - 1:
                m.nbr[e, 3] = W.BC_WALL
    return m


def _orders_fixed_y(E, Ny, seed):
    """N_y fixed (faces conforming along y), N_x, N_z random in 1..4: every
    mortar then interpolates along a direction the test data are constant in."""
    rng = np.random.default_rng(seed)
    o = rng.integers(1, 5, size=(E, 3)).astype(np.int32)
    o[:, 1] = Ny
    return o


# ----------------------------------------------------------------------------
# Q19 exact polynomial NS solutions
# ----------------------------------------------------------------------------

MU, PR = 0.05, 0.72
KAPPA = MU * GAMMA / ((GAMMA - 1.0) * PR)
A_SH, P0, B_T = 0.7, 1.3, 0.4

SOLUTIONS = {
    # u = a y^2, rho = 1, p const: d(rho u)/dt = d tau_xy/dy = 2 a mu,
    # dE/dt = d(u tau_xy)/dy = 6 a^2 mu y^2 (inviscid part zero)
    "shear": (lambda x, y, z: (1.0 + 0 * x, A_SH * y * y, 0 * x, 0 * x, P0 + 0 * x),
              lambda x, y, z: (0.0, 2 * A_SH * MU, 0.0, 0.0, 6 * A_SH ** 2 * MU * y * y)),
    # u = 0, rho = 1, p = p0 + b y^2, T = p/rho: d(rho v)/dt = -dp/dy,
    # dE/dt = d(kappa dT/dy)/dy = 2 kappa b
    "heat": (lambda x, y, z: (1.0 + 0 * x, 0 * x, 0 * x, 0 * x, P0 + B_T * y * y),
             lambda x, y, z: (0.0, 0.0, -2 * B_T * y, 0.0, 2 * KAPPA * B_T)),
}


@pytest.mark.parametrize("name", ["shear", "heat"])
def test_q19_ns_exact_solution(name, handle=None):
    prim, qdot = SOLUTIONS[name]
    m = _channel_mesh(5)
    P = O.Problem(m, O.phys(O.NS, mu=MU, Pr=PR), handle=handle)
    o = _orders_fixed_y(m.E, 5, seed=19)
    X = P.node_coords(o)
    q = _fields(X, o, prim)
    ref = _expect(X, o, qdot)
    scale = np.abs(ref).max()
    ri = P.rhs(o, q, O.ISOLATED)
    assert np.abs(ri - ref).max() < 1e-11 * max(scale, 1.0), np.abs(ri - ref).max()
    # non-isolated: BR1 face averages; elements two away from the periodic wrap in y
    rn = P.rhs(o, q)
    offq = W.offsets(o, 5)
    for e in range(m.E):
        if (e // 2) % 5 == 2:
            assert np.abs(rn[offq[e]:offq[e + 1]] - ref[offq[e]:offq[e + 1]]).max() < 1e-11 * max(scale, 1.0)


def test_q19_ns_divergence_term(handle=None):
    """u = a x^2, rho = 1, p = p0: tau_xx = mu (2 u_x - 2/3 u_x) = 8/3 mu a x,
    Qdot = (-2ax, -4a^2x^3 + 8/3 mu a, 0, 0,
            -2 gamma p0 a x/(gamma-1) - 3a^3x^5 + 8 mu a^2 x^2); N_x = 6
    differentiates the degree-6 energy flux exactly."""
    a = 0.6
    m = W.cube_mesh(2, 2, 2, L=(0.8, 0.5, 0.4))
    P = O.Problem(m, O.phys(O.NS, mu=MU, Pr=PR), handle=handle)
    o = np.tile(np.array([[6, 2, 1]], np.int32), (m.E, 1))
    X = P.node_coords(o)
    q = _fields(X, o, lambda x, y, z: (1.0 + 0 * x, a * x * x, 0 * x, 0 * x, P0 + 0 * x))
    g = GAMMA
    ref = _expect(X, o, lambda x, y, z: (-2 * a * x, -4 * a * a * x ** 3 + 8.0 / 3.0 * MU * a, 0.0, 0.0,
                                          -2 * g * P0 * a * x / (g - 1) - 3 * a ** 3 * x ** 5 + 8 * MU * a * a * x * x))
    r = P.rhs(o, q, O.ISOLATED)
    assert np.abs(r - ref).max() < 1e-11 * np.abs(ref).max(), np.abs(r - ref).max()


# ----------------------------------------------------------------------------
# Q20 viscous step bound
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("Pr", [0.72, 2.0])
def test_q20_dfl_closed_form(Pr, handle=None):
    """dt = min(CFL / max sum_d (|u.a^d| + c|a^d|)(N_d+1)^2/2,
               DFL / max sum_d nu_max |a^d|^2 (N_d+1)^4/4),
    nu_max = (mu/rho) max(4/3, gamma/Pr), |a^d| = 2/h_d on an affine box
    (reading A11).  Pr = 0.72: gamma/Pr wins; Pr = 2: 4/3 wins."""
    L = (1.0, 2.0, 0.8)
    m = W.cube_mesh(4, 4, 4, L=L)
    mu = 0.3
    P = O.Problem(m, O.phys(O.NS, mu=mu, Pr=Pr), handle=handle)
    N = (3, 4, 5)
    o = W.orders_uniform(m.E, N)
    rho, vel, p = 1.2, (1.0, -0.5, 0.25), 0.9
    q = W.uniform_state(o, rho=rho, vel=vel, p=p)
    c = math.sqrt(GAMMA * p / rho)
    h = [L[d] / 4 for d in range(3)]
    lam = sum((abs(vel[d]) + c) * (2 / h[d]) * (N[d] + 1) ** 2 / 2 for d in range(3))
    nu = mu / rho * max(4.0 / 3.0, GAMMA / Pr)
    vis = sum(nu * (2 / h[d]) ** 2 * (N[d] + 1) ** 4 / 4 for d in range(3))
    cfl, dfl = 0.5, 0.4
    ref = min(cfl / lam, dfl / vis)
    assert dfl / vis < cfl / lam  # the viscous bound decides
    assert abs(P.dt(o, q, cfl, dfl) - ref) <= 2e-15 * ref  # a few ulp (state round trip)


# ----------------------------------------------------------------------------
# Q21 wall faces: discrete flux balance in closed form
# ----------------------------------------------------------------------------

def test_q21_wall_flux_balance(handle=None):
    """Channel between no-slip adiabatic walls at y = 0 and y = 1 (reading
    A10), periodic in x and z: rho = 1, u = a y (1 - y), p = p0 + b y^2.
    Interior fluxes cancel (discrete conservation), so
      sum_nodes M Qdot = -A (F_y(top) - F_y(bottom)),   A = L_x L_z,
    with the wall flux F_y = Roe(q, mirror q) - f^nu(q, grad q) and a zero
    viscous energy flux (u = 0, adiabatic): (0, -2 mu a A, -b A, 0, 0)."""
    a, b = 0.8, 0.3
    L = (0.7, 1.0, 0.6)
    m = _channel_mesh(4, walls=True, L=L)
    P = O.Problem(m, O.phys(O.NS, mu=MU, Pr=PR), handle=handle)
    o = _orders_fixed_y(m.E, 5, seed=21)
    X = P.node_coords(o)
    q = _fields(X, o, lambda x, y, z: (1.0 + 0 * x, a * y * (1 - y), 0 * x, 0 * x, P0 + b * y * y))
    r = P.rhs(o, q)
    M = P.mass(o)
    offm = W.offsets(o, 1)
    offq = W.offsets(o, 5)
    tot = np.zeros(5)
    for e in range(m.E):
        n = offm[e + 1] - offm[e]
        tot += (r[offq[e]:offq[e + 1]].reshape(5, n) * M[offm[e]:offm[e + 1]]).sum(1)
    A = L[0] * L[2]
    ref = np.array([0.0, -2 * MU * a * A, -b * A, 0.0, 0.0])
    assert np.abs(tot - ref).max() < 1e-12, tot - ref


# ----------------------------------------------------------------------------
# Q22 BR1 gradient: discrete Gauss theorem with the face state qhat
# ----------------------------------------------------------------------------

def _face_nodes(N, d, s):
    """Own node indices of face (d, s) in tangential order (t1 fastest)."""
    n = [N[0] + 1, N[1] + 1, N[2] + 1]
    t1, t2 = [(1, 2), (0, 2), (0, 1)][d]
    out = []
    for b in range(n[t2]):
        for a in range(n[t1]):
            idx = [0, 0, 0]
            idx[d] = (n[d] - 1) if s else 0
            idx[t1], idx[t2] = a, b
            out.append(idx[0] + n[0] * (idx[1] + n[1] * idx[2]))
    return np.array(out), (t1, t2)


def test_q22_br1_gauss_identity(handle=None):
    """sum_nodes w J g_k = sum_faces +- sum_face-nodes w w qhat (J a^d)_k on
    every element (summation by parts of the GL operator: W D + D^T W = B),
    with qhat = (q_L + q_R)/2 inside, (rho, 0, 0, 0, E - |m|^2/(2 rho)) at a
    wall and (q + q_inf)/2 at the far field (reading A10).  Random
    discontinuous data, conforming faces, affine box: J a^d = (prod_{d'!=d}
    h_d'/2) e_d."""
    L = (0.9, 1.0, 0.7)
    m = _channel_mesh(3, walls=True, L=L)
    m.nbr[0, 2] = W.BC_FARFIELD  # one far-field face too
    qinf = W.conserved(np.array(1.1), np.array(0.3), np.array(-0.2), np.array(0.1), np.array(1.0))
    P = O.Problem(m, O.phys(O.NS, mu=MU, Pr=PR, qinf=qinf), handle=handle)
    N = (3, 4, 2)
    o = W.orders_uniform(m.E, N)
    rng = np.random.default_rng(22)
    offq = W.offsets(o, 5)
    n = int(np.prod(np.array(N) + 1))
    q = np.empty(offq[-1])
    for e in range(m.E):
        prim = (1 + 0.2 * rng.random(n), 0.3 * rng.standard_normal(n), 0.3 * rng.standard_normal(n),
                0.3 * rng.standard_normal(n), 1 + 0.2 * rng.random(n))
        q[offq[e]:offq[e + 1]] = W.conserved(*prim).ravel()
    grad = P.gradient(o, q)
    bas = [O.basis(N[d]) for d in range(3)]
    w3 = np.einsum("k,j,i->kji", bas[2]["w"], bas[1]["w"], bas[0]["w"]).ravel()
    h = [L[0] / 2, L[1] / 3, L[2] / 2]
    J = h[0] * h[1] * h[2] / 8
    offg = W.offsets(o, 15)
    for e in range(m.E):
        qe = q[offq[e]:offq[e + 1]].reshape(5, n)
        ge = grad[offg[e]:offg[e + 1]].reshape(3, 5, n)
        lhs = (ge * (w3 * J)).sum(-1)  # [k][v]
        rhs = np.zeros((3, 5))
        for d in range(3):
            Ja = np.prod([h[dd] / 2 for dd in range(3) if dd != d])
            for s in (0, 1):
                own, (t1, t2) = _face_nodes(N, d, s)
                wt = np.outer(bas[t2]["w"], bas[t1]["w"]).ravel()
                nb = int(m.nbr[e, 2 * d + s])
                qo = qe[:, own]
                if nb >= 0:
                    other, _ = _face_nodes(N, d, 1 - s)
                    qh = 0.5 * (qo + q[offq[nb]:offq[nb + 1]].reshape(5, n)[:, other])
                elif nb == W.BC_WALL:
                    qh = np.stack([qo[0], 0 * qo[0], 0 * qo[0], 0 * qo[0],
                                   qo[4] - 0.5 * (qo[1] ** 2 + qo[2] ** 2 + qo[3] ** 2) / qo[0]])
                else:
                    qh = 0.5 * (qo + qinf[:, None])
                rhs[d] += (1 if s else -1) * Ja * (qh * wt).sum(-1)
        assert np.abs(lhs - rhs).max() < 1e-13 * max(1.0, np.abs(rhs).max()), (e, np.abs(lhs - rhs).max())


# ----------------------------------------------------------------------------
# Q23 dynamic decrease cap
# ----------------------------------------------------------------------------

def test_q23_decrease_cap_properties(handle=None):
    """n_d <- max(n_d, N_d - cap) ("decrease by one", A16): the result
    never drops more than cap below the current order, never lowers a
    selection, is either the selection or N_d - cap, is idempotent, and
    cap >= N_max - 1 leaves every selection unchanged."""
    rng = np.random.default_rng(23)
    E = 400
    cur = rng.integers(1, 9, size=(E, 3)).astype(np.int32)
    sel = rng.integers(1, 9, size=(E, 3)).astype(np.int32)
    for cap in (1, 2, 3):
        out = O.decrease_cap(cur, sel, cap, handle=handle)
        assert np.all(out >= cur - cap)
        assert np.all(out >= sel)
        assert np.all((out == sel) | (out == cur - cap))
        assert np.array_equal(O.decrease_cap(cur, out, cap, handle=handle), out)
        # a drop of exactly cap is reachable (the cap binds where sel < cur - cap)
        binding = sel < cur - cap
        assert binding.any() and np.all(out[binding] == cur[binding] - cap)
    assert np.array_equal(O.decrease_cap(cur, sel, 7, handle=handle), sel)


# ----------------------------------------------------------------------------
# Q9 decoupling of the directional estimates (reading A12)
# ----------------------------------------------------------------------------

def _tau_field_full(P, orders, q, r, e, n):
    """tau~ of element e for a SIMULTANEOUS coarsening of all directions to
    orders n: I_n R_ref - Qdot_c(I_n q) (isolated coarse
    residual), from the oracle's transfer + isolated residual."""
    oc = orders.copy()
    oc[e] = n
    qc = O.transfer(orders, q, oc)
    rc = O.transfer(orders, r, oc)
    diff = rc - P.rhs(oc, qc, O.ISOLATED)
    offc = W.offsets(oc, 5)
    return diff[offc[e]:offc[e + 1]]


def test_q9_decoupling(handle=None):
    """Affine-flux data (u, p constant, rho a smooth pulse: f is affine in q at
    every node) on one periodic element, SAME reference: the full field
    tau~(n1,n2,n3) = sum_d (x)_{d' != d} I^{d'} tau~_d(n_d)."""
    m = W.cube_mesh(1, L=(0.6, 0.5, 0.7))
    P = O.Problem(m, handle=handle)
    N = np.array([[6, 5, 4]], np.int32)
    X = P.node_coords(N)
    q = W.pulse_state(X, N, center=(0.31, 0.27, 0.4), sigma=0.2, L=(0.6, 0.5, 0.7))
    r = P.rhs(N, q, O.ISOLATED)
    for n in ([3, 2, 2], [5, 4, 1], [2, 3, 3]):
        n = np.array(n, np.int32)
        full = _tau_field_full(P, N, q, r, 0, n)
        acc = np.zeros_like(full)
        for d in range(3):
            od = N.copy()
            od[0, d] = n[d]
            td = P.tau_field(N, q, r, 0, d, int(n[d])).ravel()  # field at orders od
            acc += O.transfer(od, td, n[None, :])
        assert np.abs(full - acc).max() < 1e-11 * np.abs(full).max(), np.abs(full - acc).max()  # rounding ~2e-12
        assert np.abs(full).max() > 1e-6  # a non-trivial field
