"""Multi-rank driver: one process per GPU, torch.distributed (NCCL over
NVLink/NVSwitch on GPUs, gloo on CPU for tests) for the halo exchange and
the global reductions; every numerical step runs in libdgtau's kernels.

Per residual evaluation (RK stage, SOLVER reference) one halo exchange of
partition-boundary FACE TRACES of the state with the face-neighbour ranks
(NS: a second one of the gradient's face traces after the BR1 pass) --
packed and unpacked on the device by dg_trace_copy, sent with NCCL P2P
(partition.TracePlan; a rank's halo elements only ever have their faces
toward owned elements read); per RK step one MAX
all-reduce of the CFL/DFL rates (dt = CFL / global max, reading A11); per
jump-fixpoint sweep one exchange of halo orders and one MAX all-reduce of the
`changed` flag (the fixpoint is monotone, so the result is rank-count
invariant).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import partition as part


def exchange(tensor, plan: "part.HaloPlan", rank: int, group=None):
    """Refresh halo ranges of `tensor` (1-D) from the owning ranks.  Contiguous
    runs are sent as views (no packing when a run covers a peer's range)."""
    import torch
    import torch.distributed as dist

    ops, bufs = [], []
    for r in sorted(plan.send):
        sruns, rruns = plan.send[r], plan.recv[r]
        if len(sruns) == 1:
            sbuf = tensor[sruns[0][0]:sruns[0][1]]
        else:
            sbuf = torch.cat([tensor[a:b] for a, b in sruns])
        if len(rruns) == 1:
            rbuf = tensor[rruns[0][0]:rruns[0][1]]
        else:
            rbuf = torch.empty(plan.recv_len[r], dtype=tensor.dtype, device=tensor.device)
            bufs.append((rbuf, rruns))
        ops.append(dist.P2POp(dist.isend, sbuf.contiguous(), r, group))
        ops.append(dist.P2POp(dist.irecv, rbuf, r, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for rbuf, rruns in bufs:
        o = 0
        for a, b in rruns:
            tensor[a:b].copy_(rbuf[o:o + b - a])
            o += b - a


class TraceExchange:
    """Device-side face-trace exchange of one field (state: ncomp 5, or the
    BR1 gradient: ncomp 15) for a DistSolver's current layout: per peer rank
    the entry tables (partition.TracePlan) on the device and persistent
    send / receive buffers."""

    def __init__(self, S, plan: "part.TracePlan"):
        import torch

        self.S, self.plan = S, plan
        dev = torch.device("cuda", torch.cuda.current_device())
        self.send = {r: torch.from_numpy(t).to(dev) for r, t in plan.send.items()}
        self.recv = {r: torch.from_numpy(t).to(dev) for r, t in plan.recv.items()}
        self.sbuf = {r: torch.empty(max(1, plan.send_len[r]), dtype=torch.float64, device=dev) for r in plan.send}
        self.rbuf = {r: torch.empty(max(1, plan.recv_len[r]), dtype=torch.float64, device=dev) for r in plan.recv}

    def bytes_per_exchange(self):
        return 8 * sum(self.plan.send_len.values())

    def start(self, field, group=None):
        """pack on the current stream and post the P2P operations (NCCL runs
        them on its own stream once the packs are done); returns the requests"""
        import torch.distributed as dist

        nc = self.plan.ncomp
        ops = []
        for r in sorted(self.send):
            self.S.trace_copy(self.send[r], field, nc, self.sbuf[r], 0)
            ops.append(dist.P2POp(dist.isend, self.sbuf[r][: max(1, self.plan.send_len[r])], r, group))
            ops.append(dist.P2POp(dist.irecv, self.rbuf[r][: max(1, self.plan.recv_len[r])], r, group))
        return dist.batch_isend_irecv(ops) if ops else []

    def finish(self, field, reqs):
        """the current stream waits for the transfers, then unpacks"""
        for req in reqs:
            req.wait()
        nc = self.plan.ncomp
        for r in sorted(self.recv):
            self.S.trace_copy(self.recv[r], field, nc, self.rbuf[r], 1)

    def __call__(self, field, group=None):
        self.finish(field, self.start(field, group))


def migrate(q_owned, plan: "part.MigrationPlan", group=None):
    """Move owned element states to their new owners after a repartition
    (SURVEY 8(f) rank 2): one all_to_all_single (NCCL on GPUs, gloo on CPU).
    q_owned: 1-D states of plan.old_ids (increasing global id); returns the
    states of plan.new_ids (increasing global id)."""
    import torch
    import torch.distributed as dist

    dev = q_owned.device
    pos = {int(g): i for i, g in enumerate(plan.old_ids)}
    chunks = []
    for ids in plan.send_ids:
        for g in ids:
            i = pos[int(g)]
            chunks.append(q_owned[int(plan.old_off[i]):int(plan.old_off[i + 1])])
    send = torch.cat(chunks) if chunks else torch.empty(0, dtype=q_owned.dtype, device=dev)
    recv = torch.empty(sum(plan.recv_len), dtype=q_owned.dtype, device=dev)
    dist.all_to_all_single(recv, send, plan.recv_len, plan.send_len, group=group)
    # received blocks come grouped by source rank; order them by global id
    src = np.concatenate([ids for ids in plan.recv_ids]) if plan.recv_ids else np.zeros(0, np.int64)
    lens = plan.n[src]
    starts = np.concatenate([[0], np.cumsum(lens)])
    order = np.argsort(src, kind="stable")
    out = torch.empty_like(recv)
    o = 0
    for k in order:
        a, b = int(starts[k]), int(starts[k + 1])
        out[o:o + b - a].copy_(recv[a:b])
        o += b - a
    return out


def gather_layout(own_gids, world, group=None, device="cuda"):
    """(counts, max count, global row index of every gathered row in rank
    order): the owned global element ids of every rank, gathered once per
    local mesh."""
    import torch
    import torch.distributed as dist

    gathered = [None] * world
    dist.all_gather_object(gathered, np.asarray(own_gids, np.int64), group=group)
    counts = [len(g) for g in gathered]
    return counts, max(counts), torch.from_numpy(np.concatenate(gathered)).to(device)


def gather_rows(own_rows, layout, world, group=None):
    """Global [sum(counts), k] tensor from every rank's owned rows [n_own, k]
    (row i of rank r lands at its global id): one all_gather of equal-sized
    padded blocks, 4k bytes per element, on the rows' device."""
    import torch
    import torch.distributed as dist

    counts, nmax, gidx = layout
    k = own_rows.shape[1]
    send = torch.zeros((nmax, k), dtype=own_rows.dtype, device=own_rows.device)
    send[: own_rows.shape[0]] = own_rows
    recv = torch.empty((world * nmax, k), dtype=own_rows.dtype, device=own_rows.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    res = torch.empty((sum(counts), k), dtype=own_rows.dtype, device=own_rows.device)
    res[gidx] = torch.cat([recv[r * nmax: r * nmax + counts[r]] for r in range(world)])
    return res


class DistSolver:
    """A `Solver` on this rank's local mesh (owned + halo elements) plus the
    exchanges that make owned results identical to the single-rank ones."""

    def __init__(self, global_mesh, owner: np.ndarray, rank: int, world: int, group=None, overlap=False,
                 **solver_kw):
        """overlap: each RK stage launches the faces without a halo side while
        the halo traces are in flight (runtime-order path: curved meshes, or
        path=PATH_RUNTIME on affine ones)."""
        from . import Solver

        self.rank, self.world, self.group, self.overlap = rank, world, group, overlap
        self.mesh, self.owner, self.solver_kw = global_mesh, np.asarray(owner), dict(solver_kw)
        self.lm = part.local_mesh(global_mesh, owner, rank)
        self.physics = solver_kw.get("physics", 0)
        self.S = Solver(self.lm, **solver_kw)
        self.S._check(self.S.L.dg_set_owned(self.S.ctx, int(self.lm.n_own)), "dg_set_owned")
        self.plan = None
        self.gplan = None
        import torch

        self._lam = torch.zeros(2, dtype=torch.int64, device="cuda")

    # -- layout ------------------------------------------------------------
    def set_orders(self, global_orders):
        lo = np.ascontiguousarray(np.asarray(global_orders)[self.lm.gids], np.int32)
        self.S.set_orders(lo)
        self.local_orders = lo
        self.plan = part.HaloPlan(self.lm, lo, 5)  # whole element states (rebalancing refresh)
        self.tq = TraceExchange(self.S, part.TracePlan(self.lm, lo, 5))
        self._level_tx = {}  # non-isolated tau levels: gradient trace exchanges of the coarse layouts
        self.tg = TraceExchange(self.S, part.TracePlan(self.lm, lo, 15)) if self.physics == 1 else None

    @property
    def n_own(self):
        return self.lm.n_own

    def owned_len(self):
        return int(self.S.L.dg_owned_state_len(self.S.ctx))

    def new_state(self):
        return self.S.new_state()

    def halo(self, q):
        """face traces of the state toward owned elements (what the residual reads)"""
        self.tq(q, self.group)

    def halo_states(self, q):
        """whole element states of the halo (after a repartition)"""
        exchange(q, self.plan, self.rank, self.group)

    # -- operators -----------------------------------------------------------
    def _gradient_halo(self, q, variant=0):
        """NS: BR1 gradients of the owned elements, then their halo refresh
        (the viscous face flux needs the neighbour's gradient trace)."""
        from . import FLAG_GRADIENT_READY, NS

        if self.physics != NS:
            return 0
        self.S.gradient(q, variant)
        if variant == 0:
            self.tg(self.S.gradient_buffer(), self.group)
        return FLAG_GRADIENT_READY

    def rhs_eval(self, q, qdot=None, variant=0):
        if variant == 0:
            self.halo(q)
        flags = self._gradient_halo(q, variant)
        qdot = self.S.new_state() if qdot is None else qdot
        self.S._check(self.S.L.dg_rhs_eval_flags(self.S.ctx, int(variant), C.c_void_p(q.data_ptr()),
                                                 C.c_void_p(qdot.data_ptr()), int(flags), self._stream()),
                      "dg_rhs_eval_flags")
        return qdot

    def compute_dt(self, q, cfl, dt):
        import torch.distributed as dist

        self._lam.zero_()
        self.S._check(self.S.L.dg_dt_accumulate(self.S.ctx, C.c_void_p(q.data_ptr()),
                                                C.c_void_p(self._lam.data_ptr()), self._stream()), "dg_dt_accumulate")
        dist.all_reduce(self._lam, op=dist.ReduceOp.MAX, group=self.group)
        self.S._check(self.S.L.dg_dt_finalize(self.S.ctx, C.c_void_p(self._lam.data_ptr()), C.c_double(cfl),
                                              C.c_void_p(dt.data_ptr()), self._stream()), "dg_dt_finalize")
        return dt

    def _stream(self):
        import torch

        return C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def rk_step_dt(self, q_in, q_out, g, dt, cfl, dt_next):
        """Three stages with a halo refresh before each; the CFL rates of the
        new state are reduced in the last stage and MAX-all-reduced."""
        import torch.distributed as dist

        src, dst = [q_in, q_out, q_in], [q_out, q_in, q_out]
        self._lam.zero_()
        for k in range(3):
            if self.overlap:
                self._stage_overlapped(k, src[k], dst[k], g, dt)
                continue
            self.halo(src[k])
            flags = self._gradient_halo(src[k])
            self.S.rk_stage(k, src[k], dst[k], g, dt, self._lam if k == 2 else None, flags)
        dist.all_reduce(self._lam, op=dist.ReduceOp.MAX, group=self.group)
        self.S._check(self.S.L.dg_dt_finalize(self.S.ctx, C.c_void_p(self._lam.data_ptr()), C.c_double(cfl),
                                              C.c_void_p(dt_next.data_ptr()), self._stream()), "dg_dt_finalize")

    def _stage_overlapped(self, k, q, q_out, g, dt):
        """One RK stage with the trace exchanges overlapped: the faces with no
        halo side run while the traces are in flight; the halo
        faces and the element kernels after the exchange completes."""
        from . import FLAG_FACES_HALO, FLAG_FACES_INTERIOR, FLAG_GRADIENT_READY, NS

        lam = self._lam if k == 2 else None
        reqs = self.tq.start(q, self.group)
        if self.physics == NS:
            self.S.gradient(q, flags=FLAG_FACES_INTERIOR)
            self.tq.finish(q, reqs)
            self.S.gradient(q, flags=FLAG_FACES_HALO)
            gb = self.S.gradient_buffer()
            reqs = self.tg.start(gb, self.group)
            self.S.rk_stage(k, q, q_out, g, dt, lam, FLAG_GRADIENT_READY | FLAG_FACES_INTERIOR)
            self.tg.finish(gb, reqs)
            self.S.rk_stage(k, q, q_out, g, dt, lam, FLAG_GRADIENT_READY | FLAG_FACES_HALO)
        else:
            self.S.rk_stage(k, q, q_out, g, dt, lam, FLAG_FACES_INTERIOR)
            self.tq.finish(q, reqs)
            self.S.rk_stage(k, q, q_out, g, dt, lam, FLAG_FACES_HALO)

    def tau_estimate(self, q, qdot_ref=None, noniso=False, **kw):
        """Isolated levels: element-local.  noniso (SURVEY 8(f) rank 1,
        P:217-219): every coarse level (d, p) of the global loop (MAX
        all-reduce of the orders) in two phases, the level's BR1 gradient face
        traces exchanged between them (NS); the halo's coarse state traces
        follow from the fine ones already exchanged."""
        if noniso and kw.get("restriction", 0) != 0:
            raise NotImplementedError("non-isolated tau across ranks: the L2-projection restriction reads halo "
                                      "interiors; use the interpolation restriction (reading A3)")
        tau = self.S.tau_estimate(q, qdot_ref, **kw)  # slot 0 and the undefined entries; levels overwrite the rest
        if not noniso:
            return tau
        import torch
        import torch.distributed as dist

        n_own = self.lm.n_own
        nmax = torch.tensor(self.local_orders[:n_own].max(axis=0), dtype=torch.int64, device="cuda")
        dist.all_reduce(nmax, op=dist.ReduceOp.MAX, group=self.group)
        form = kw.get("formulation", 0)
        restr = kw.get("restriction", 0)
        for d in range(3):
            for p in range(1, int(nmax[d].item())):
                lev = self.S.tau_level(d, p, 0, q, qdot_ref, formulation=form, restriction=restr)
                if self.physics == 1:
                    key = (d, p)
                    if key not in self._level_tx:
                        oc = self.local_orders.copy()
                        oc[:, d] = np.minimum(oc[:, d], p)
                        self._level_tx[key] = TraceExchange(lev, part.TracePlan(self.lm, oc, 15))
                    tx = self._level_tx[key]
                    tx.S = lev
                    tx(lev.gradient_buffer(), self.group)
                self.S.tau_level(d, p, 1, tau=tau, formulation=form, restriction=restr)
        return tau

    def select_orders(self, tau, tau_max, Nmin, Nmax, rule=1, dec_cap=1, mode=0, total_map=None):
        """Map/select/cap on owned elements, then the jump fixpoint with halo
        order exchanges; returns the global orders array (all ranks)."""
        import torch
        import torch.distributed as dist

        from . import _Policy

        pol = _Policy(int(mode), float(tau_max), int(Nmin), int(Nmax), int(rule), int(dec_cap))
        E = self.lm.E
        a = torch.empty((E, 3), dtype=torch.int32, device="cuda")
        b = torch.empty_like(a)
        S = self.S
        S._check(S.L.dg_select_local(S.ctx, C.byref(pol), C.c_void_p(tau.data_ptr()),
                                     C.c_void_p(0 if total_map is None else total_map.data_ptr()),
                                     C.c_void_p(a.data_ptr()), None, self._stream()), "dg_select_local")
        if getattr(self, "_oplan", None) is None:  # depends on the local mesh only
            self._oplan = part.HaloPlan(self.lm, np.zeros((E, 3), np.int32), 3)  # 3 ints per element, n = 1 node
        oplan = self._oplan
        changed = torch.zeros(1, dtype=torch.int32, device="cuda")
        for _ in range(64):
            flat = a.view(-1)
            exchange(flat, oplan, self.rank, self.group)
            changed.zero_()
            S._check(S.L.dg_jump_sweep(S.ctx, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), int(rule), int(Nmax),
                                       C.c_void_p(changed.data_ptr()), self._stream()), "dg_jump_sweep")
            a, b = b, a
            dist.all_reduce(changed, op=dist.ReduceOp.MAX, group=self.group)
            if int(changed.item()) == 0:
                break
        n_own = self.lm.n_own
        # NCCL: device to device; gloo (CPU tests): the same gather on host tensors
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        if getattr(self, "_gather_layout", None) is None:  # once per local mesh
            self._gather_layout = gather_layout(self.lm.gids[:n_own], self.world, self.group, dev)
        return gather_rows(a[:n_own].to(dev), self._gather_layout, self.world, self.group).cpu().numpy()


def rebalance(ds: DistSolver, global_orders, q_local, axis: int = 2):
    """Dynamic load rebalancing after an adaptation: a new
    DOF-balanced slab partition for `global_orders` (partition.dof_owner), the
    owned element states moved with one all-to-all (migrate), a new DistSolver
    on the new local mesh, and its halo refreshed.  q_local: this rank's local
    state (owned + halo) at global_orders under the old partition.  Returns
    (new DistSolver, new local state)."""
    import torch

    go = np.asarray(global_orders, np.int32)
    new_owner = part.dof_owner(ds.mesh.dims, go, ds.world, axis)
    plan = part.MigrationPlan(ds.owner, new_owner, go, ds.rank, ds.world)
    q_own = migrate(q_local[: int(plan.old_off[-1])], plan, ds.group)
    nd = DistSolver(ds.mesh, new_owner, ds.rank, ds.world, ds.group, overlap=ds.overlap, **ds.solver_kw)
    nd.set_orders(go)
    n = part.element_offsets(go[nd.lm.gids])
    q_new = torch.zeros(int(n[-1]), dtype=q_local.dtype, device=q_local.device)
    q_new[: q_own.numel()].copy_(q_own)
    nd.halo_states(q_new)
    return nd, q_new
