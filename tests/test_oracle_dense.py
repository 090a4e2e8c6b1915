"""Q24 (SURVEY 8(c).3 row "Q17 ultra-brute"): the oracle's sum-factorised
residual against a DENSE Galerkin assembly on 4-8-element meshes (CPU, -m
"not gpu").

The dense side is the weak form of P:119-140 (eqs DGSEMsystem:1-2) written out
with no tensor-product structure: every trial function phi_m = l_i l_j l_k and
its gradient is evaluated at every quadrature point by the Lagrange product
formulas (no Kronecker deltas, no derivative matrix), the element integrals
and the face integrals are plain sums over the Gauss-Lobatto points

    M_m qdot_m =  sum_n W_n J  F(q_n) . grad phi_m(xi_n)
                - sum_faces sum_s w_s JA  F*(q-, q+; n) phi_m(xi_s),

the face values q-, q+ are the element polynomials evaluated at the face
points, the GL rule comes from numpy's Legendre module, and the Euler flux
and the local Lax-Friedrichs flux (the A7 flag, P:472 names Roe; LLF is the
oracle's second solver) are retyped here in numpy.  Strong and weak forms are
equal on GL points (summation by parts), so the oracle must agree to
rounding, whichever form it uses.  For Navier-Stokes the BR1 gradient
(P:137-140 eq DGSEMsystem:2, qhat = average) is assembled densely the same
way and the viscous flux f^nu(q, g) is the oracle's point function, pinned by
hand values in Q3 and by the exact solutions of Q19: this pin fixes the
ASSEMBLY (indices, metric factors 2/h_d, face orientation, signs, lifting
weights) on anisotropic orders, for both systems.
"""
import numpy as np
import pytest
from numpy.polynomial import legendre as L

import oracle as O
import workloads as W

GAMMA = 1.4


def _gl(N):
    """Gauss-Lobatto points / weights of order N from Legendre polynomials:
    the roots of P_N' and +-1, w = 2 / (N (N+1) P_N(x)^2)."""
    c = np.zeros(N + 1)
    c[N] = 1.0
    x = np.concatenate(([-1.0], np.sort(L.legroots(L.legder(c)).real), [1.0])) if N > 1 else np.array([-1.0, 1.0])
    w = 2.0 / (N * (N + 1) * L.legval(x, c) ** 2)
    return x, w


def _lag(xs, i, x):
    return np.prod([(x - xs[r]) / (xs[i] - xs[r]) for r in range(len(xs)) if r != i])


def _dlag(xs, i, x):
    s = 0.0
    for t in range(len(xs)):
        if t == i:
            continue
        s += 1.0 / (xs[i] - xs[t]) * np.prod([(x - xs[r]) / (xs[i] - xs[r]) for r in range(len(xs)) if r not in (i, t)])
    return s


def _euler(q, d):
    rho, m, E = q[0], q[1:4], q[4]
    u = m / rho
    p = (GAMMA - 1.0) * (E - 0.5 * (m * u).sum(0))
    f = np.stack([m[d], m[0] * u[d], m[1] * u[d], m[2] * u[d], (E + p) * u[d]])
    f[1 + d] += p
    return f


def _llf(qL, qR, d, sgn):
    """Rusanov flux along the outward normal sgn * e_d."""
    def un_c(q):
        u = q[1 + d] / q[0] * sgn
        p = (GAMMA - 1.0) * (q[4] - 0.5 * (q[1:4] ** 2).sum(0) / q[0])
        return u, np.sqrt(GAMMA * p / q[0])
    uL, cL = un_c(qL)
    uR, cR = un_c(qR)
    lam = np.maximum(np.abs(uL) + cL, np.abs(uR) + cR)
    return 0.5 * sgn * (_euler(qL, d) + _euler(qR, d)) - 0.5 * lam * (qR - qL)


class _Dense:
    """Dense tables of one order triple: trial functions and their reference
    gradients at all volume points, and trial functions at all face points."""

    def __init__(self, N):
        self.N = N
        self.r = [_gl(n) for n in N]
        xs = [r[0] for r in self.r]
        n1, n2, n3 = (n + 1 for n in N)
        self.n = n1 * n2 * n3
        idx = [(i, j, k) for k in range(n3) for j in range(n2) for i in range(n1)]   # i fastest
        self.idx = idx
        self.Wt = np.array([self.r[0][1][i] * self.r[1][1][j] * self.r[2][1][k] for i, j, k in idx])
        self.G = np.zeros((3, self.n, self.n))     # G[d][m, n] = d phi_m / d xi_d at point n
        for m, (i, j, k) in enumerate(idx):
            for n, (a, b, c) in enumerate(idx):
                pt = (xs[0][a], xs[1][b], xs[2][c])
                l = (_lag(xs[0], i, pt[0]), _lag(xs[1], j, pt[1]), _lag(xs[2], k, pt[2]))
                dl = (_dlag(xs[0], i, pt[0]), _dlag(xs[1], j, pt[1]), _dlag(xs[2], k, pt[2]))
                self.G[0][m, n] = dl[0] * l[1] * l[2]
                self.G[1][m, n] = l[0] * dl[1] * l[2]
                self.G[2][m, n] = l[0] * l[1] * dl[2]
        # faces f = 2 d + s: points (t1, t2) over the two other directions, lower direction fastest
        self.B, self.wf = [], []
        for f in range(6):
            d, s = divmod(f, 2)
            o = [t for t in range(3) if t != d]
            pts, wts = [], []
            for b2 in range(N[o[1]] + 1):
                for b1 in range(N[o[0]] + 1):
                    p = [0.0, 0.0, 0.0]
                    p[d] = -1.0 if s == 0 else 1.0
                    p[o[0]] = xs[o[0]][b1]
                    p[o[1]] = xs[o[1]][b2]
                    pts.append(p)
                    wts.append(self.r[o[0]][1][b1] * self.r[o[1]][1][b2])
            B = np.array([[_lag(xs[0], i, p[0]) * _lag(xs[1], j, p[1]) * _lag(xs[2], k, p[2]) for p in pts]
                          for (i, j, k) in idx])          # B[m, s]
            self.B.append(B)
            self.wf.append(np.array(wts))


def _dense_rhs(mesh, N, q, ph=None):
    """Qdot (and the BR1 gradient for NS) of a conforming periodic affine box
    with the same order triple N in every element."""
    T = _Dense(N)
    E, n = mesh.E, T.n
    h = mesh.extra["h"]
    J = h[0] * h[1] * h[2] / 8.0
    Mm = J * T.Wt
    Q = q.reshape(E, 5, n)
    ns = ph is not None
    # face traces of every element (dense evaluation of the polynomial at the face points)
    tr = [[Q[e] @ T.B[f] for f in range(6)] for e in range(E)]
    g = np.zeros((E, 3, 5, n))
    if ns:
        for e in range(E):
            for d in range(3):
                acc = -(Q[e] * (T.Wt * J * 2.0 / h[d])) @ T.G[d].T                 # - sum_n W J q_n d_d phi_m
                for s in range(2):
                    f = 2 * d + s
                    qh = 0.5 * (tr[e][f] + tr[mesh.nbr[e, f]][f ^ 1])
                    acc += (qh * (T.wf[f] * J * 2.0 / h[d] * (1.0 if s else -1.0))) @ T.B[f].T
                g[e, d] = acc / Mm
    gtr = [[np.stack([g[e, d] @ T.B[f] for d in range(3)]) for f in range(6)] for e in range(E)] if ns else None

    def fvisc(qp, gp, d):
        out = np.empty_like(qp)
        for s in range(qp.shape[1]):
            out[:, s] = O.viscous_flux(qp[:, s], gp[:, :, s].ravel(), d, ph)
        return out

    out = np.empty((E, 5, n))
    for e in range(E):
        acc = np.zeros((5, n))
        for d in range(3):
            F = _euler(Q[e], d)
            if ns:
                F = F - fvisc(Q[e], g[e], d)
            acc += (F * (T.Wt * J * 2.0 / h[d])) @ T.G[d].T
            for s in range(2):
                f = 2 * d + s
                nb = mesh.nbr[e, f]
                sgn = 1.0 if s else -1.0
                Fs = _llf(tr[e][f], tr[nb][f ^ 1], d, sgn)
                if ns:
                    Fs = Fs - 0.5 * sgn * (fvisc(tr[e][f], gtr[e][f], d) + fvisc(tr[nb][f ^ 1], gtr[nb][f ^ 1], d))
                acc -= (Fs * (T.wf[f] * J * 2.0 / h[d])) @ T.B[f].T
        out[e] = acc / Mm
    return out.ravel(), g


def _state(prob, orders, seed):
    X = prob.node_coords(orders)
    E = len(orders)
    n = X.size // (3 * E)
    x, y, z = X.reshape(E, 3, n).transpose(1, 0, 2)
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.05, 0.15, 5)
    two_pi = 2.0 * np.pi
    rho = 1.0 + a[0] * np.sin(two_pi * x) * np.cos(two_pi * y) + a[1] * np.sin(two_pi * z)
    u = 0.8 + a[2] * np.cos(two_pi * (x + y))
    v = -0.3 + a[3] * np.sin(two_pi * (y - z))
    w = 0.2 + a[4] * np.cos(two_pi * x) * np.sin(two_pi * z)
    p = 1.0 + 0.1 * np.sin(two_pi * (x + z))
    q = W.conserved(rho, u, v, w, p)                 # [5][E][n]
    return np.ascontiguousarray(np.asarray(q).transpose(1, 0, 2)).ravel()


@pytest.mark.parametrize("dims,N", [((2, 2, 1), (3, 2, 4)), ((2, 2, 2), (2, 3, 1)), ((1, 2, 2), (5, 1, 2))])
def test_q24_dense_euler(dims, N, handle=None):
    mesh = W.cube_mesh(*dims, L=(1.0, 0.8, 1.3))
    orders = W.orders_uniform(mesh.E, N)
    prob = O.Problem(mesh, O.phys(O.EULER, O.LLF, GAMMA), handle=handle)
    q = _state(prob, orders, 11)
    ref, _ = _dense_rhs(mesh, N, q)
    got = prob.rhs(orders, q)
    assert np.abs(got - ref).max() < 1e-12 * np.abs(ref).max()
    # the dense form sees a dropped term: it is not small
    assert np.abs(ref).max() > 1.0


@pytest.mark.parametrize("dims,N", [((2, 2, 1), (3, 2, 4)), ((2, 1, 2), (2, 4, 3))])
def test_q24_dense_navier_stokes(dims, N, handle=None):
    mesh = W.cube_mesh(*dims, L=(1.0, 0.8, 1.3))
    orders = W.orders_uniform(mesh.E, N)
    ph = O.phys(O.NS, O.LLF, GAMMA, mu=0.05, Pr=0.72)
    prob = O.Problem(mesh, ph, handle=handle)
    q = _state(prob, orders, 12)
    ref, g = _dense_rhs(mesh, N, q, ph)
    gg = prob.gradient(orders, q).reshape(g.shape)
    assert np.abs(gg - g).max() < 1e-12 * np.abs(g).max()
    got = prob.rhs(orders, q)
    assert np.abs(got - ref).max() < 1e-12 * np.abs(ref).max()
    # the viscous part is visible at this mu: the Euler residual differs by far more than the bar
    eul = O.Problem(mesh, O.phys(O.EULER, O.LLF, GAMMA)).rhs(orders, q)
    assert np.abs(eul - ref).max() > 1e-3 * np.abs(ref).max()


# ----------------------------------------------------------------------------
# Q25 Roe flux on general subsonic states (reading A7: no entropy fix)
# ----------------------------------------------------------------------------

def _roe(handle, qL, qR, n):
    if handle is None:
        return O.roe_flux(qL, qR, n, GAMMA)
    import ctypes as C
    F = np.empty(5)
    handle.orc_roe_flux(*(C.c_void_p(a.ctypes.data) for a in (qL, qR, n)), C.c_double(GAMMA), C.c_void_p(F.ctypes.data))
    return F


def test_q25_roe_matrix_absolute_value(handle=None):
    """Roe's solver is F = 1/2 (f_L + f_R).n - 1/2 |A~| (q_R - q_L), A~ the
    flux Jacobian d(f.n)/dq at the Roe-averaged velocity and total enthalpy
    (the Jacobian is homogeneous of degree 0: it depends on u and H only).
    Here A~ is the complex-step derivative of the numpy Euler flux and |A~| =
    sqrt(A~ A~) the principal matrix square root (scipy): no eigenvectors,
    no wave strengths.  Also Roe's property A~ dq = df, which pins the
    averaging itself."""
    from scipy.linalg import sqrtm
    rng = np.random.default_rng(25)

    def fn(q, n):
        return sum(n[k] * _euler(q, k) for k in range(3))

    worst = 0.0
    for _ in range(200):
        prim = lambda: (rng.uniform(0.5, 2.0), rng.uniform(-0.6, 0.6, 3), rng.uniform(0.7, 2.0))  # noqa: E731
        (rL, uL, pL), (rR, uR, pR) = prim(), prim()
        qL = np.array([rL, *(rL * uL), pL / (GAMMA - 1) + 0.5 * rL * uL @ uL])
        qR = np.array([rR, *(rR * uR), pR / (GAMMA - 1) + 0.5 * rR * uR @ uR])
        n = rng.normal(size=3)
        n /= np.linalg.norm(n)
        sl, sr = np.sqrt(rL), np.sqrt(rR)
        u = (sl * uL + sr * uR) / (sl + sr)
        H = (sl * (qL[4] + pL) / rL + sr * (qR[4] + pR) / rR) / (sl + sr)
        if abs(u @ n) < 0.02:      # |A| is not smooth at a vanishing eigenvalue: stay off it
            continue
        qt = np.array([1.0, *u, (H + 0.5 * (GAMMA - 1) * u @ u) / GAMMA])
        A = np.empty((5, 5))
        for j in range(5):
            qc = qt.astype(complex)
            qc[j] += 1e-30j
            A[:, j] = fn(qc, n).imag / 1e-30
        assert np.abs(A @ (qR - qL) - (fn(qR, n) - fn(qL, n))).max() < 1e-13     # Roe's property
        absA = sqrtm(A @ A).real
        ref = 0.5 * (fn(qL, n) + fn(qR, n)) - 0.5 * absA @ (qR - qL)
        got = _roe(handle, qL, qR, n)
        worst = max(worst, np.abs(got - ref).max() / np.abs(ref).max())
    assert worst < 1e-11
