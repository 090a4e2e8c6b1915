"""B200-native (sm_100a) hot path of tau-estimation-driven anisotropic
p-adaptation for the DGSEM (arXiv 2210.03523).

Thin Python binding over the C ABI in ``include/dgtau.h`` (``libdgtau.so``,
built in-tree by :func:`build`).  Argument marshalling only: every numerical
step runs in the library's CUDA kernels.  PyTorch provides device memory and
streams.  There is no CPU fallback: importing works without a GPU (so the
CPU test-suite can check the exported symbols), but every compute call
raises if the library or a CUDA device is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libdgtau.so")
_CSRC = os.path.join(_HERE, "csrc")
_INC = os.path.join(os.path.dirname(_HERE), "include")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]

EULER, NS = 0, 1
ROE, LLF = 0, 1
NONISOLATED, ISOLATED = 0, 1
TAU_NEW, TAU_TRADITIONAL = 0, 1
PATH_AUTO, PATH_RUNTIME, PATH_BUCKETED = 0, 1, 2
REF_SOLVER, REF_SAME = 0, 1
JUMP_A, JUMP_B = 0, 1
SELECT_DYNAMIC, SELECT_STATIC_ACCUM, SELECT_STATIC_FINAL, SELECT_A1_ACCUM, SELECT_A1_FINAL = 0, 1, 2, 3, 4
COMBINE_MAX, COMBINE_AV = 0, 1
TAU_STRIDE = 9
FLAG_GRADIENT_READY = 1
FLAG_FACES_INTERIOR, FLAG_FACES_HALO = 2, 4
NMAX = 8

EXPORTS = ["dg_create", "dg_destroy", "dg_last_error", "dg_mesh_upload", "dg_set_orders", "dg_state_len", "dg_ndof",
           "dg_node_coords", "dg_rhs_eval", "dg_compute_dt", "dg_rk_step", "dg_tau_estimate", "dg_select_orders",
           "dg_transfer", "dg_diagnostics", "dg_launch_count", "dg_rk_step_dt", "dg_set_owned", "dg_rk_stage",
           "dg_dt_accumulate", "dg_dt_finalize", "dg_select_local", "dg_jump_sweep", "dg_owned_state_len", "dg_gradient",
           "dg_gradient_buffer", "dg_rhs_eval_flags", "dg_rk_steps", "dg_trace_copy", "dg_tau_level", "dg_set_path", "dg_gradient_flags"]


def sources():
    return [os.path.join(_CSRC, f) for f in sorted(os.listdir(_CSRC)) if f.endswith((".cu", ".cpp", ".cuh", ".h"))] + \
        [os.path.join(_INC, "dgtau.h")]


def _digest(srcs):
    import hashlib

    h = hashlib.sha1()
    for s in srcs:
        h.update(os.path.basename(s).encode())
        h.update(open(s, "rb").read())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libdgtau.so for sm_100a with nvcc (cross-compiles without a GPU).
    Skipped when the library's stamp matches the sources' content hash."""
    import fcntl

    srcs = sources()
    stamp = _SO + ".stamp"
    dig = _digest(srcs)
    with open(_SO + ".lock", "w") as lk:  # the ranks of a torchrun job call this at once: one compiles
        fcntl.flock(lk, fcntl.LOCK_EX)
        fresh = os.path.exists(_SO) and os.path.exists(stamp) and open(stamp).read().strip() == dig
        if force or not fresh:
            _compile(srcs, verbose)
            with open(stamp, "w") as f:
                f.write(dig)
    return _SO


def _compile(srcs, verbose=False, force_all=False):
    """Objects in parallel (res_inst.cu once per N1 = 1..8: the 512
    order-specialised residual kernels dominate), then link."""
    from concurrent.futures import ThreadPoolExecutor

    objdir = os.path.join(_HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    units = []
    for s in srcs:
        if os.path.basename(s) == "res_inst.cu":
            units += [(s, [f"-DRES_N1={k}"], f"res_inst_{k}.cu.o") for k in range(1, 9)]
        elif s.endswith((".cu", ".cpp")):
            units.append((s, [], os.path.basename(s) + ".o"))
    hdr_t = max(os.path.getmtime(s) for s in srcs if s.endswith((".cuh", ".h")))
    # the 512 order-specialised residual instances include residual_t.cuh only
    res_t = max(os.path.getmtime(os.path.join(_CSRC, h)) for h in ("residual_t.cuh", "common.cuh", "basis.h"))
    cflags = [f for f in NVCC_FLAGS if f != "-shared"]

    def one(u):
        src, defs, name = u
        obj = os.path.join(objdir, name)
        dep_t = res_t if defs else hdr_t
        if not force_all and os.path.exists(obj) and os.path.getmtime(obj) > max(os.path.getmtime(src), dep_t):
            return obj
        cmd = ["nvcc", *cflags, *defs, "-c", src, "-o", obj] + (["-Xptxas=-v"] if verbose else [])
        subprocess.check_call(cmd)
        return obj

    with ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(one, units))
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", _SO, *objs])


class DGError(RuntimeError):
    pass


class _Params(C.Structure):
    _fields_ = [("physics", C.c_int), ("flux", C.c_int), ("gamma", C.c_double), ("mu", C.c_double),
                ("Pr", C.c_double), ("qinf", C.c_double * 5)]


class _TauOpts(C.Structure):
    _fields_ = [("formulation", C.c_int), ("reference", C.c_int), ("coarse_faces", C.c_int), ("restriction", C.c_int)]


class _Policy(C.Structure):
    _fields_ = [("mode", C.c_int), ("tau_max", C.c_double), ("Nmin", C.c_int), ("Nmax", C.c_int),
                ("jump_rule", C.c_int), ("dec_cap", C.c_int), ("combine", C.c_int), ("nstages", C.c_int)]


_lib = None


def lib():
    """Load libdgtau.so; raises if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        so = os.environ.get("DGTAU_SO", _SO)  # A/B timing of in-tree kernel variants (tools/)
        if not os.path.exists(so):
            raise DGError(f"{so} not built: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(so)
        L.dg_last_error.restype = C.c_char_p
        L.dg_state_len.restype = C.c_int64
        L.dg_ndof.restype = C.c_int64
        L.dg_launch_count.restype = C.c_int64
        L.dg_owned_state_len.restype = C.c_int64
        L.dg_gradient_buffer.restype = C.c_void_p
        for name in EXPORTS:
            getattr(L, name)
        _lib = L
    return _lib


def _device_view(ptr, n):
    """Borrowed fp64 CUDA tensor over context-owned memory (lifetime: the context)."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 2}

    return torch.as_tensor(_Arr(), device="cuda")


def _ptr(t):
    """device pointer of a torch tensor (or None), unchecked (context-owned views)."""
    return C.c_void_p(0 if t is None else t.data_ptr())


def _dptr(t, n, what, dtype=None, optional=False):
    """Checked device pointer for the C ABI: a contiguous CUDA tensor of the
    expected dtype (float64 by default) with at least n elements.  The kernels
    trust the pointer and the layout, so a wrong tensor is rejected here
    instead of being read out of bounds on the GPU."""
    import torch

    if t is None:
        if optional:
            return C.c_void_p(0)
        raise DGError(f"{what}: tensor required")
    dt = torch.float64 if dtype is None else dtype
    if not isinstance(t, torch.Tensor):
        raise DGError(f"{what}: expected a torch tensor, got {type(t).__name__}")
    if t.dtype != dt:
        raise DGError(f"{what}: dtype {t.dtype}, expected {dt}")
    if not t.is_cuda:
        raise DGError(f"{what}: tensor must live on the CUDA device")
    if not t.is_contiguous():
        raise DGError(f"{what}: tensor must be contiguous")
    if t.numel() < n:
        raise DGError(f"{what}: {t.numel()} elements, needs at least {n}")
    return C.c_void_p(t.data_ptr())


def _np(a, dtype):
    return np.ascontiguousarray(a, dtype)


def _stream(stream):
    import torch

    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


class Level:
    """Borrowed handle of a non-isolated tau level's context (owned by its
    parent Solver's context; valid until the parent's next set_orders)."""

    def __init__(self, L, ctx, state_len):
        self.L, self.ctx, self.state_len = L, ctx, state_len

    def _check(self, rc, what):
        if rc != 0:
            raise DGError(f"{what} failed ({rc}): {self.L.dg_last_error(self.ctx).decode()}")

    def gradient_buffer(self):
        ptr = self.L.dg_gradient_buffer(self.ctx)
        if not ptr:
            raise DGError("level: no gradient buffer")
        return _device_view(ptr, 3 * self.state_len)

    def trace_copy(self, entries, field, ncomp, buf, direction, stream=None):
        import torch

        n = int(entries.shape[0])
        self._check(self.L.dg_trace_copy(self.ctx, _dptr(entries, 2 * n, "trace entries", torch.int64), n,
                                         _dptr(field, (ncomp // 5) * self.state_len, "trace field"), int(ncomp),
                                         _dptr(buf, 0, "trace buffer"), int(direction), _stream(stream)),
                    "dg_trace_copy")


class Solver:
    """One DGSEM discretisation on the current CUDA device.

    mesh: object with ``nbr`` [E][6] int32, ``gorder`` (3,), ``geo`` [E][3][ng]
    (see workloads.Mesh).  State tensors are fp64 CUDA tensors in the
    canonical layout of include/dgtau.h.
    """

    def __init__(self, mesh, physics=EULER, flux=ROE, gamma=1.4, mu=0.0, Pr=0.72, qinf=None, path=PATH_AUTO):
        """path: PATH_AUTO, or PATH_RUNTIME (runtime-order kernels on affine
        meshes too: many-bucket layouts under dynamic adaptation; dg_set_path)."""
        import torch

        if not torch.cuda.is_available():
            raise DGError("no CUDA device: the DGSEM path runs only on the GPU (no CPU fallback)")
        self.L = lib()
        p = _Params()
        p.physics, p.flux, p.gamma, p.mu, p.Pr = physics, flux, gamma, mu, Pr
        qi = np.zeros(5) if qinf is None else np.asarray(qinf, np.float64)
        for v in range(5):
            p.qinf[v] = qi[v]
        self.ctx = C.c_void_p()
        torch.cuda.current_device()
        self._check(self.L.dg_create(C.byref(p), C.byref(self.ctx)), "dg_create")
        if path != PATH_AUTO:
            self._check(self.L.dg_set_path(self.ctx, int(path)), "dg_set_path")
        self.nbr = _np(mesh.nbr, np.int32)
        self.E = int(self.nbr.shape[0])
        gord = _np(mesh.gorder, np.int32)
        geo = _np(mesh.geo, np.float64)
        self._check(self.L.dg_mesh_upload(self.ctx, self.E, self.nbr.ctypes.data_as(C.c_void_p),
                                          gord.ctypes.data_as(C.c_void_p), geo.ctypes.data_as(C.c_void_p)),
                    "dg_mesh_upload")
        self.orders = None
        self._dt = torch.zeros(1, dtype=torch.float64, device="cuda")

    def _check(self, rc, what):
        if rc != 0:
            msg = self.L.dg_last_error(self.ctx).decode() if self.ctx else ""
            raise DGError(f"{what} failed ({rc}): {msg}")

    def __del__(self):
        try:
            if self.ctx:
                self.L.dg_destroy(self.ctx)
        except Exception:
            pass

    # -- layout ----------------------------------------------------------
    def set_orders(self, orders):
        o = _np(orders, np.int32)
        self._check(self.L.dg_set_orders(self.ctx, o.ctypes.data_as(C.c_void_p)), "dg_set_orders")
        self.orders = o.copy()

    @property
    def state_len(self) -> int:
        return int(self.L.dg_state_len(self.ctx))

    @property
    def ndof(self) -> int:
        return int(self.L.dg_ndof(self.ctx))

    @property
    def launches(self) -> int:
        return int(self.L.dg_launch_count(self.ctx))

    def node_coords(self):
        X = np.empty(3 * self.ndof)
        self._check(self.L.dg_node_coords(self.ctx, X.ctypes.data_as(C.c_void_p)), "dg_node_coords")
        return X

    def new_state(self):
        import torch

        return torch.empty(self.state_len, dtype=torch.float64, device="cuda")

    # -- operators --------------------------------------------------------
    def rhs_eval(self, q, qdot=None, variant=NONISOLATED, stream=None):
        qdot = self.new_state() if qdot is None else qdot
        n = self.state_len
        self._check(self.L.dg_rhs_eval(self.ctx, int(variant), _dptr(q, n, "rhs_eval q"), _dptr(qdot, n, "rhs_eval qdot"),
                                       _stream(stream)), "dg_rhs_eval")
        return qdot

    def compute_dt(self, q, cfl, dt=None, sync=False, stream=None):
        dt = self._dt if dt is None else dt
        host = C.c_double(0.0)
        self._check(self.L.dg_compute_dt(self.ctx, _dptr(q, self.state_len, "compute_dt q"), C.c_double(cfl),
                                         _dptr(dt, 1, "compute_dt dt"),
                                         C.byref(host) if sync else None, _stream(stream)), "dg_compute_dt")
        return host.value if sync else dt

    def rk_step(self, q_in, q_out, g, dt, stream=None):
        n = self.state_len
        self._check(self.L.dg_rk_step(self.ctx, _dptr(q_in, n, "rk_step q_in"), _dptr(q_out, n, "rk_step q_out"),
                                      _dptr(g, n, "rk_step g"), _dptr(dt, 1, "rk_step dt"), _stream(stream)),
                    "dg_rk_step")

    def rk_step_dt(self, q_in, q_out, g, dt, cfl, dt_next, stream=None):
        """RK3 step; the CFL dt of the new state is reduced inside the last stage."""
        n = self.state_len
        self._check(self.L.dg_rk_step_dt(self.ctx, _dptr(q_in, n, "rk_step_dt q_in"), _dptr(q_out, n, "rk_step_dt q_out"),
                                         _dptr(g, n, "rk_step_dt g"), _dptr(dt, 1, "rk_step_dt dt"), C.c_double(cfl),
                                         _dptr(dt_next, 1, "rk_step_dt dt_next"), _stream(stream)), "dg_rk_step_dt")

    def rk_steps(self, nsteps, qa, qb, g, dt_a, dt_b, cfl, stream=None):
        """nsteps RK3 steps ping-ponging (qa, qb) and (dt_a, dt_b) on the device
        (dg_rk_steps); returns (state, next dt) tensors after the last step."""
        n = self.state_len
        self._check(self.L.dg_rk_steps(self.ctx, int(nsteps), _dptr(qa, n, "rk_steps qa"), _dptr(qb, n, "rk_steps qb"),
                                       _dptr(g, n, "rk_steps g"), _dptr(dt_a, 1, "rk_steps dt_a"),
                                       _dptr(dt_b, 1, "rk_steps dt_b"), C.c_double(cfl), _stream(stream)), "dg_rk_steps")
        return (qa, dt_a) if nsteps % 2 == 0 else (qb, dt_b)

    # -- multi-rank pieces (see dist.py) ---------------------------------------
    def set_owned(self, n_owned):
        self._check(self.L.dg_set_owned(self.ctx, int(n_owned)), "dg_set_owned")

    def owned_len(self):
        return int(self.L.dg_owned_state_len(self.ctx))

    def rk_stage(self, k, q_in, q_out, g, dt, lam=None, flags=0, stream=None):
        import torch

        n = self.state_len
        self._check(self.L.dg_rk_stage(self.ctx, int(k), _dptr(q_in, n, "rk_stage q_in"), _dptr(q_out, n, "rk_stage q_out"),
                                       _dptr(g, n, "rk_stage g"), _dptr(dt, 1, "rk_stage dt"),
                                       _dptr(lam, 2, "rk_stage lam", torch.int64, optional=True), int(flags),
                                       _stream(stream)), "dg_rk_stage")

    def gradient(self, q, variant=NONISOLATED, stream=None, flags=0):
        """BR1 gradient into gradient_buffer(); flags FLAG_FACES_INTERIOR /
        FLAG_FACES_HALO split its face pass around a halo exchange."""
        self._check(self.L.dg_gradient_flags(self.ctx, int(variant), _dptr(q, self.state_len, "gradient q"), int(flags),
                                             _stream(stream)), "dg_gradient_flags")

    def gradient_buffer(self):
        """torch view of the context's gradient buffer (15 doubles per node)."""
        import torch

        n = 3 * self.state_len
        ptr = self.L.dg_gradient_buffer(self.ctx)
        if not ptr:
            raise DGError("no gradient buffer (NS on the curved path only)")
        return _device_view(ptr, n)

    def dt_accumulate(self, q, lam, stream=None):
        self._check(self.L.dg_dt_accumulate(self.ctx, _ptr(q), _ptr(lam), _stream(stream)), "dg_dt_accumulate")

    def dt_finalize(self, lam, cfl, dt, stream=None):
        self._check(self.L.dg_dt_finalize(self.ctx, _ptr(lam), C.c_double(cfl), _ptr(dt), _stream(stream)),
                    "dg_dt_finalize")

    def select_local(self, tau, tau_max, Nmin, Nmax, out, mode=SELECT_DYNAMIC, dec_cap=1, total_map=None, stream=None):
        pol = _Policy(int(mode), float(tau_max), int(Nmin), int(Nmax), JUMP_B, int(dec_cap), COMBINE_MAX, 0)
        self._check(self.L.dg_select_local(self.ctx, C.byref(pol), _ptr(tau), _ptr(total_map), _ptr(out), None,
                                           _stream(stream)), "dg_select_local")

    def trace_copy(self, entries, field, ncomp, buf, direction, stream=None):
        """Pack (direction 0: field -> buf) or unpack (1: buf -> face nodes of
        field) partition-boundary face traces (partition.TracePlan entries,
        int64 [n][2] on the device)."""
        import torch

        n = int(entries.shape[0])
        self._check(self.L.dg_trace_copy(self.ctx, _dptr(entries, 2 * n, "trace entries", torch.int64), n,
                                         _dptr(field, (ncomp // 5) * self.state_len, "trace field"), int(ncomp),
                                         _dptr(buf, 0, "trace buffer"), int(direction), _stream(stream)),
                    "dg_trace_copy")

    def jump_sweep(self, a, b, rule, Nmax, changed, stream=None):
        self._check(self.L.dg_jump_sweep(self.ctx, _ptr(a), _ptr(b), int(rule), int(Nmax), _ptr(changed),
                                         _stream(stream)), "dg_jump_sweep")

    def tau_estimate(self, q, qdot_ref=None, formulation=TAU_NEW, reference=REF_SOLVER, tau=None, stream=None,
                     noniso=False, restriction=0):
        """tau[e][d][p].  noniso=True: non-isolated coarse residuals
        (whole mesh at each level's coarse orders; single rank).
        restriction: 0 interpolation (A3), 1 exact L2 projection (A3 flag)."""
        import torch

        o = _TauOpts(int(formulation), int(reference), 1 if noniso else 0, int(restriction))
        tau = torch.empty((self.E, 3, TAU_STRIDE), dtype=torch.float64, device="cuda") if tau is None else tau
        n = self.state_len
        self._check(self.L.dg_tau_estimate(self.ctx, C.byref(o), _dptr(q, n, "tau_estimate q"),
                                           _dptr(qdot_ref, n, "tau_estimate qdot_ref", optional=reference == REF_SAME),
                                           _dptr(tau, self.E * 3 * TAU_STRIDE, "tau_estimate tau"), _stream(stream)),
                    "dg_tau_estimate")
        return tau

    def tau_level(self, d, p, phase, q=None, qdot_ref=None, tau=None, formulation=TAU_NEW, restriction=0, stream=None):
        """One non-isolated tau level (d, p) in two phases (dg_tau_level, for
        rank-local meshes): phase 0 -> Level handle (its BR1 gradient formed;
        refresh its halo face traces), phase 1 writes tau[e][d][p]."""
        o = _TauOpts(int(formulation), REF_SOLVER, 1, int(restriction))
        lev = C.c_void_p()
        n = self.state_len
        self._check(self.L.dg_tau_level(self.ctx, int(d), int(p), int(phase), C.byref(o),
                                        _dptr(q, n, "tau_level q", optional=phase == 1),
                                        _dptr(qdot_ref, n, "tau_level qdot_ref", optional=phase == 1),
                                        _dptr(tau, self.E * 3 * TAU_STRIDE, "tau_level tau", optional=phase == 0),
                                        C.byref(lev), _stream(stream)), "dg_tau_level")
        return Level(self.L, lev, int(self.L.dg_state_len(lev)))

    def select_orders(self, tau, tau_max, Nmin, Nmax, mode=SELECT_DYNAMIC, jump_rule=JUMP_B, dec_cap=1,
                      total_map=None, stream=None, combine=COMBINE_MAX, nstages=0):
        """Orders from tau.  Static approach 2 (SELECT_STATIC_*,
        total_map [E][K][K][K]) or approach 1 (SELECT_A1_*, total_map [E][3]);
        combine F_max / F_av (nstages = n_e for the F_av finals)."""
        pol = _Policy(int(mode), float(tau_max), int(Nmin), int(Nmax), int(jump_rule), int(dec_cap), int(combine),
                      int(nstages))
        out = np.zeros((self.E, 3), np.int32)
        margin = np.zeros(self.E)
        self._check(self.L.dg_select_orders(self.ctx, C.byref(pol), _dptr(tau, self.E * 3 * TAU_STRIDE, "select tau"),
                                            _ptr(total_map),
                                            out.ctypes.data_as(C.c_void_p), margin.ctypes.data_as(C.c_void_p),
                                            _stream(stream)), "dg_select_orders")
        return out, margin

    def transfer(self, new_orders, q_old, out=None, stream=None):
        """State projected onto new_orders.  `out`: optional device
        buffer of at least the new state length (reused, no allocation)."""
        import torch

        no = _np(new_orders, np.int32)
        n = int((5 * np.prod(no.astype(np.int64) + 1, axis=1)).sum())
        if out is not None:
            if out.numel() < n:
                raise DGError(f"transfer: out has {out.numel()} doubles, needs {n}")
            q_new = out[:n]
        else:
            q_new = torch.empty(n, dtype=torch.float64, device="cuda")
        self._check(self.L.dg_transfer(self.ctx, no.ctypes.data_as(C.c_void_p), _dptr(q_old, self.state_len, "transfer q_old"),
                                       _dptr(q_new, n, "transfer q_new"),
                                       _stream(stream)), "dg_transfer")
        return q_new

    def diagnostics(self, q, v=None, stream=None):
        sums = np.zeros(5)
        mn = np.zeros(2)
        self._check(self.L.dg_diagnostics(self.ctx, _dptr(q, self.state_len, "diagnostics q"),
                                          _dptr(v, self.state_len, "diagnostics v", optional=True),
                                          sums.ctypes.data_as(C.c_void_p),
                                          mn.ctypes.data_as(C.c_void_p), _stream(stream)), "dg_diagnostics")
        return sums, mn
