"""Python face of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2210_03523_b200`` never imports it.

Thin ctypes marshalling around ``liboracle.so`` (built from
``dgsem_oracle.c`` by :func:`build`); all arithmetic lives in the C file,
whose functions cite PAPER.md line by line.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "dgsem_oracle.c")

EULER, NS = 0, 1
ROE, LLF = 0, 1
NONISOLATED, ISOLATED = 0, 1
TAU_NEW, TAU_TRADITIONAL = 0, 1
JUMP_A, JUMP_B = 0, 1
TAU_STRIDE = 9
SENTINEL = 1e30
NMAX = 16


def build(force: bool = False) -> str:
    import hashlib

    hdr = os.path.join(_HERE, "dgsem_oracle.h")
    dig = hashlib.sha1(open(_SRC, "rb").read() + open(hdr, "rb").read()).hexdigest()
    stamp = _SO + ".stamp"
    fresh = os.path.exists(_SO) and os.path.exists(stamp) and open(stamp).read().strip() == dig
    if force or not fresh:
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"])
        with open(stamp, "w") as f:
            f.write(dig)
    return _SO


class _Phys(C.Structure):
    _fields_ = [("gamma", C.c_double), ("physics", C.c_int), ("flux", C.c_int),
                ("mu", C.c_double), ("Pr", C.c_double), ("qinf", C.c_double * 5)]


class _Mesh(C.Structure):
    _fields_ = [("E", C.c_int), ("nbr", C.c_void_p), ("gorder", C.c_void_p), ("geo", C.c_void_p)]


_lib = None


def load(path: str):
    """ctypes handle of an oracle library at ``path`` (the built one by
    default; tests load mutated copies to show that the pins catch them)."""
    h = C.CDLL(path)
    h.orc_compute_dt.restype = C.c_double
    return h


def lib():
    global _lib
    if _lib is None:
        _lib = load(build())
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data)


def phys(physics=EULER, flux=ROE, gamma=1.4, mu=0.0, Pr=0.72, qinf=None):
    ph = _Phys()
    ph.gamma = gamma
    ph.physics = physics
    ph.flux = flux
    ph.mu = mu
    ph.Pr = Pr
    qi = np.zeros(5) if qinf is None else np.asarray(qinf, np.float64)
    for v in range(5):
        ph.qinf[v] = qi[v]
    return ph


class Problem:
    """Holds the mesh arrays alive for the C side."""

    def __init__(self, mesh, ph=None, handle=None):
        self.nbr = np.ascontiguousarray(mesh.nbr, np.int32)
        self.gorder = np.ascontiguousarray(mesh.gorder, np.int32)
        self.geo = np.ascontiguousarray(mesh.geo, np.float64)
        self.E = int(self.nbr.shape[0])
        self.m = _Mesh(self.E, _p(self.nbr).value, _p(self.gorder).value, _p(self.geo).value)
        self.ph = ph if ph is not None else phys()
        self._h = handle

    def L(self):
        return self._h if self._h is not None else lib()

    # -- helpers -------------------------------------------------------
    @staticmethod
    def _ord(orders):
        return np.ascontiguousarray(orders, np.int32)

    @staticmethod
    def size(orders, ncomp=5):
        return int(ncomp * np.prod(np.asarray(orders, np.int64) + 1, axis=1).sum())

    # -- operators -----------------------------------------------------
    def node_coords(self, orders):
        o = self._ord(orders)
        X = np.empty(self.size(o, 3))
        self.L().orc_node_coords(C.byref(self.m), _p(o), _p(X))
        return X

    def mass(self, orders):
        o = self._ord(orders)
        M = np.empty(self.size(o, 1))
        self.L().orc_mass(C.byref(self.m), _p(o), _p(M))
        return M

    def rhs(self, orders, q, variant=NONISOLATED):
        o = self._ord(orders)
        q = np.ascontiguousarray(q, np.float64)
        out = np.empty_like(q)
        rc = self.L().orc_rhs(C.byref(self.m), _p(o), _p(q), int(variant), C.byref(self.ph), _p(out))
        if rc:
            raise ValueError("orc_rhs failed")
        return out

    def gradient(self, orders, q, variant=NONISOLATED):
        o = self._ord(orders)
        q = np.ascontiguousarray(q, np.float64)
        out = np.empty(self.size(o, 15))
        self.L().orc_gradient(C.byref(self.m), _p(o), _p(q), int(variant), C.byref(self.ph), _p(out))
        return out

    def dt(self, orders, q, cfl, dfl=None):
        o = self._ord(orders)
        q = np.ascontiguousarray(q, np.float64)
        return self.L().orc_compute_dt(C.byref(self.m), _p(o), _p(q), C.byref(self.ph), C.c_double(cfl),
                                    C.c_double(cfl if dfl is None else dfl))

    def rk3_step(self, orders, q, dt):
        o = self._ord(orders)
        q = np.array(q, np.float64, copy=True)
        rc = self.L().orc_rk3_step(C.byref(self.m), _p(o), _p(q), C.c_double(dt), C.byref(self.ph))
        if rc:
            raise ValueError("orc_rk3_step failed")
        return q

    def tau_estimate(self, orders, q, qdot_ref, formulation=TAU_NEW, restriction=0):
        """Isolated tau-estimation; restriction 0 = interpolation (A3), 1 = L2 projection."""
        o = self._ord(orders)
        q = np.ascontiguousarray(q, np.float64)
        r = np.ascontiguousarray(qdot_ref, np.float64)
        tau = np.empty((self.E, 3, TAU_STRIDE))
        self.L().orc_tau_estimate_r(C.byref(self.m), _p(o), _p(q), _p(r), int(formulation), int(restriction),
                                 C.byref(self.ph), _p(tau))
        return tau

    def tau_estimate_noniso(self, orders, q, qdot_ref, formulation=TAU_NEW, restriction=0):
        """NON-ISOLATED tau-estimation ("uses all terms appearing in
        the discrete DG variational formulation"; reading R7
        for the neighbours' orders).  For direction d and level p:
          O(e) = N(e) with O_d = min(p, N_d(e))        (the whole mesh at level (d, p))
          q_c = I q, R_c = I Qdot_ref                  (per-direction interpolation, A3)
          Qdot_c = non-isolated residual of the mesh at O   (Roe faces / mortars, eq DGSEMsystem)
          tau~ = R_c - Qdot_c (new form); traditional: J w w w tau~
          tau[e][d][p] = max over nodes, variables of |tau| for p < N_d(e)
        Slot 0 holds ||Qdot_ref,e||_inf (reading R1).  Composition of the oracle's
        own residual, transfer and mass operators, one level at a time."""
        o = self._ord(orders)
        q = np.ascontiguousarray(q, np.float64)
        r = np.ascontiguousarray(qdot_ref, np.float64)
        E = self.E
        tau = np.full((E, 3, TAU_STRIDE), np.nan)
        n = np.prod(o.astype(np.int64) + 1, axis=1)
        off = np.concatenate([[0], np.cumsum(5 * n)])
        for e in range(E):
            tau[e, :, 0] = np.abs(r[off[e]:off[e + 1]]).max()
        for d in range(3):
            for p in range(1, int(o[:, d].max())):
                oc = o.copy()
                oc[:, d] = np.minimum(o[:, d], p)
                if restriction:
                    qc = restrict_l2(o, q, oc, d)
                    rc = restrict_l2(o, r, oc, d)
                else:
                    qc = transfer(o, q, oc)
                    rc = transfer(o, r, oc)
                diff = rc - self.rhs(oc, qc, NONISOLATED)
                nc = np.prod(oc.astype(np.int64) + 1, axis=1)
                offc = np.concatenate([[0], np.cumsum(5 * nc)])
                scale = self.mass(oc) if formulation == TAU_TRADITIONAL else None
                offm = np.concatenate([[0], np.cumsum(nc)])
                for e in range(E):
                    if p >= o[e, d]:
                        continue
                    de = diff[offc[e]:offc[e + 1]].reshape(5, nc[e])
                    if scale is not None:
                        de = de * scale[offm[e]:offm[e + 1]][None, :]
                    tau[e, d, p] = np.abs(de).max()
        return tau

    def tau_field(self, orders, q, qdot_ref, e, d, p, formulation=TAU_NEW):
        o = self._ord(orders)
        q = np.ascontiguousarray(q, np.float64)
        r = np.ascontiguousarray(qdot_ref, np.float64)
        out = np.empty(5 * 17 ** 3)
        nc = self.L().orc_tau_field(C.byref(self.m), _p(o), _p(q), _p(r), int(e), int(d), int(p), int(formulation),
                                 C.byref(self.ph), _p(out))
        return out[: 5 * nc].reshape(5, nc)


# -- basis ---------------------------------------------------------------

def basis(N):
    x = np.empty(N + 1); w = np.empty(N + 1)
    D = np.empty((N + 1) * (N + 1)); Dh = np.empty((N + 1) * (N + 1))
    lm = np.empty(N + 1); lp = np.empty(N + 1)
    if lib().orc_basis(int(N), _p(x), _p(w), _p(D), _p(Dh), _p(lm), _p(lp)):
        raise ValueError(N)
    return dict(x=x, w=w, D=D.reshape(N + 1, N + 1), Dhat=Dh.reshape(N + 1, N + 1), lm1=lm, lp1=lp)


def interp_matrix(Nf, Nt):
    T = np.empty((Nt + 1) * (Nf + 1))
    lib().orc_interp_matrix(int(Nf), int(Nt), _p(T))
    return T.reshape(Nt + 1, Nf + 1)


def projection_matrix(M, s):
    P = np.empty((s + 1) * (M + 1))
    lib().orc_projection_matrix(int(M), int(s), _p(P))
    return P.reshape(s + 1, M + 1)


# -- point fluxes ----------------------------------------------------------

def euler_flux(q, k, gamma=1.4):
    q = np.ascontiguousarray(q, np.float64); f = np.empty(5)
    lib().orc_euler_flux(_p(q), int(k), C.c_double(gamma), _p(f))
    return f


def roe_flux(qL, qR, n, gamma=1.4):
    qL = np.ascontiguousarray(qL, np.float64); qR = np.ascontiguousarray(qR, np.float64)
    n = np.ascontiguousarray(n, np.float64); F = np.empty(5)
    lib().orc_roe_flux(_p(qL), _p(qR), _p(n), C.c_double(gamma), _p(F))
    return F


def llf_flux(qL, qR, n, gamma=1.4):
    qL = np.ascontiguousarray(qL, np.float64); qR = np.ascontiguousarray(qR, np.float64)
    n = np.ascontiguousarray(n, np.float64); F = np.empty(5)
    lib().orc_llf_flux(_p(qL), _p(qR), _p(n), C.c_double(gamma), _p(F))
    return F


def viscous_flux(q, g, k, ph):
    q = np.ascontiguousarray(q, np.float64); g = np.ascontiguousarray(g, np.float64); f = np.empty(5)
    lib().orc_viscous_flux(_p(q), _p(g), int(k), C.byref(ph), _p(f))
    return f


# -- map / selection / jump / transfer --------------------------------------

def build_map(orders, tau, Nmin, Nmax):
    o = np.ascontiguousarray(orders, np.int32)
    tau = np.ascontiguousarray(tau, np.float64)
    E = o.shape[0]; K = Nmax - Nmin + 1
    mp = np.empty((E, K, K, K)); sl = np.empty((E, 3))
    if lib().orc_build_map(E, _p(o), _p(tau), int(Nmin), int(Nmax), _p(mp), _p(sl)):
        raise ValueError("bad order range")
    return mp, sl  # mp[e, n3, n2, n1]


def combine_max(total, mp):
    total = np.ascontiguousarray(total, np.float64)
    mp = np.ascontiguousarray(mp, np.float64)
    lib().orc_combine_max(C.c_size_t(total.size), _p(total), _p(mp))
    return total


def combine_sum(total, mp):
    """Approach 2 with F_av: the total map is the mean of the stage
    maps; this accumulates its numerator (the final selection divides by n_e)."""
    return np.ascontiguousarray(total, np.float64) + np.ascontiguousarray(mp, np.float64)


def combine_degrees(picks, how=0):
    """Approach 1: N_i^e = F(N_i^{e,1}, ..., N_i^{e,n_e}) per element
    and direction, F_max (how=0) or F_av (how=1); the F_av mean is
    rounded half up (reading R8).  picks: [n_e][E][3]."""
    p = np.asarray(picks, np.float64)
    if how == 0:
        return p.max(axis=0).astype(np.int32)
    return np.floor(p.sum(axis=0) / p.shape[0] + 0.5).astype(np.int32)


def select_from_map(mp, Nmin, Nmax, tau_max):
    mp = np.ascontiguousarray(mp, np.float64)
    E = mp.shape[0]
    out = np.empty((E, 3), np.int32); mg = np.empty(E)
    lib().orc_select_from_map(E, _p(mp), int(Nmin), int(Nmax), C.c_double(tau_max), _p(out), _p(mg))
    return out, mg


def decrease_cap(cur, sel, cap=1, handle=None):
    cur = np.ascontiguousarray(cur, np.int32); sel = np.array(sel, np.int32, copy=True)
    (handle or lib()).orc_decrease_cap(cur.shape[0], _p(cur), int(cap), _p(sel))
    return sel


def jump_fixpoint(nbr, orders, rule, Nmax):
    nbr = np.ascontiguousarray(nbr, np.int32); o = np.array(orders, np.int32, copy=True)
    sweeps = lib().orc_jump_fixpoint(o.shape[0], _p(nbr), int(rule), int(Nmax), _p(o))
    return o, sweeps


def transfer(old_orders, q, new_orders, ncomp=5):
    oo = np.ascontiguousarray(old_orders, np.int32); on = np.ascontiguousarray(new_orders, np.int32)
    q = np.ascontiguousarray(q, np.float64)
    out = np.empty(Problem.size(on, ncomp))
    lib().orc_transfer(oo.shape[0], _p(oo), _p(q), _p(on), _p(out), int(ncomp))
    return out


def restrict_l2(old_orders, q, new_orders, d, ncomp=5):
    """Exact L2 projection along direction d (the A3 flag): every element's
    [v][k][j][i] block times P^{N_d -> O_d} (projection_matrix) along axis d;
    elements whose order does not change are copied."""
    oo = np.asarray(old_orders); on = np.asarray(new_orders)
    offo = np.concatenate([[0], np.cumsum(ncomp * np.prod(oo.astype(np.int64) + 1, axis=1))])
    offn = np.concatenate([[0], np.cumsum(ncomp * np.prod(on.astype(np.int64) + 1, axis=1))])
    out = np.empty(offn[-1])
    for e in range(len(oo)):
        a = oo[e] + 1
        blk = np.asarray(q[offo[e]:offo[e + 1]]).reshape(ncomp, a[2], a[1], a[0])
        if on[e, d] != oo[e, d]:
            Pm = projection_matrix(int(oo[e, d]), int(on[e, d]))  # [(s+1), (M+1)]
            ax = 3 - d  # axis of direction d in [v][k][j][i]
            blk = np.moveaxis(np.tensordot(Pm, blk, axes=([1], [ax])), 0, ax)
        out[offn[e]:offn[e + 1]] = blk.ravel()
    return out


def select_dynamic(orders, tau, nbr, tau_max, Nmin, Nmax, rule=JUMP_B, cap=1):
    """Dynamic adaptation stage (Fig. 1; cap P:672; jump P:511-520)."""
    mp, _ = build_map(orders, tau, Nmin, Nmax)
    sel, mg = select_from_map(mp, Nmin, Nmax, tau_max)
    sel = decrease_cap(orders, sel, cap)
    sel, _ = jump_fixpoint(nbr, sel, rule, Nmax)
    return sel, mg
