"""Element partitioning and halo plans for multi-rank runs.

Host logic only (O(E) index bookkeeping, no method arithmetic).  Each rank
holds a *local mesh*: its owned elements first (increasing global id), then
halo copies of the other ranks' elements that share a face with an owned
element, grouped by owning rank (increasing rank, then global id).  The
residual of an owned element needs only its own state and its face
neighbours' traces, so refreshing the halo states once per residual
evaluation reproduces the single-rank result exactly (the kernels read the
same values in the same order).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

OUTSIDE = -3  # neighbour code for faces of halo elements that leave the local set


def slab_owner(dims, world: int, axis: int = 2) -> np.ndarray:
    """Owner rank of every element of a lexicographic (i fastest) structured
    mesh with dims (n0, n1, n2): contiguous slabs along `axis`, as equal as
    possible.  axis=2 gives contiguous global-id ranges."""
    n0, n1, n2 = dims
    E = n0 * n1 * n2
    idx = np.arange(E)
    coord = [idx % n0, (idx // n0) % n1, idx // (n0 * n1)][axis]
    n = dims[axis]
    if world > n:
        raise ValueError(f"cannot split {n} element layers over {world} ranks")
    bounds = [(r * n) // world for r in range(world + 1)]
    owner = np.empty(E, np.int32)
    for r in range(world):
        owner[(coord >= bounds[r]) & (coord < bounds[r + 1])] = r
    return owner


def dof_owner(dims, orders: np.ndarray, world: int, axis: int = 2) -> np.ndarray:
    """Repartition after a p-adaptation: contiguous slabs
    of element layers along `axis` whose DOF counts are as equal as the layer
    granularity allows.  Cut r is placed at the layer boundary whose
    cumulative DOF is closest to r/world of the total (ties: the earlier
    boundary), every rank keeps at least one layer."""
    n0, n1, n2 = dims
    E = n0 * n1 * n2
    idx = np.arange(E)
    coord = [idx % n0, (idx // n0) % n1, idx // (n0 * n1)][axis]
    n = dims[axis]
    if world > n:
        raise ValueError(f"cannot split {n} element layers over {world} ranks")
    dof = np.prod(np.asarray(orders, np.int64) + 1, axis=1)
    cum = np.concatenate([[0], np.cumsum(np.bincount(coord, weights=dof, minlength=n))])
    bounds = [0]
    for r in range(1, world):
        lo, hi = bounds[-1] + 1, n - (world - r)  # at least one layer each side
        target = cum[-1] * r / world
        b = lo + int(np.argmin(np.abs(cum[lo:hi + 1] - target)))
        bounds.append(b)
    bounds.append(n)
    owner = np.empty(E, np.int32)
    for r in range(world):
        owner[(coord >= bounds[r]) & (coord < bounds[r + 1])] = r
    return owner


@dataclass
class LocalMesh:
    rank: int
    world: int
    gids: np.ndarray          # local id -> global id (owned then halo)
    n_own: int
    nbr: np.ndarray           # [E_loc][6] local ids, BC codes, or OUTSIDE
    gorder: tuple
    geo: np.ndarray
    send: dict = field(default_factory=dict)  # rank -> local ids of owned elements to send (ordered)
    recv: dict = field(default_factory=dict)  # rank -> local ids of halo elements to receive (ordered)
    kind: str = "affine"

    @property
    def E(self) -> int:
        return int(self.gids.shape[0])


def local_mesh(mesh, owner: np.ndarray, rank: int) -> LocalMesh:
    world = int(owner.max()) + 1
    nbr_g = np.asarray(mesh.nbr)
    owned = np.flatnonzero(owner == rank)
    own_set = np.zeros(len(owner), bool)
    own_set[owned] = True
    nb = nbr_g[owned].ravel()
    nb = nb[nb >= 0]
    halo = np.unique(nb[~own_set[nb]])
    halo = halo[np.lexsort((halo, owner[halo]))]  # by owning rank, then global id
    gids = np.concatenate([owned, halo]).astype(np.int64)
    g2l = -np.ones(len(owner), np.int64)
    g2l[gids] = np.arange(len(gids))
    loc = nbr_g[gids].astype(np.int64)
    mapped = np.where(loc >= 0, g2l[np.maximum(loc, 0)], loc)
    mapped = np.where((loc >= 0) & (mapped < 0), OUTSIDE, mapped)
    lm = LocalMesh(rank=rank, world=world, gids=gids, n_own=len(owned), nbr=mapped.astype(np.int32),
                   gorder=tuple(mesh.gorder), geo=np.ascontiguousarray(np.asarray(mesh.geo)[gids]),
                   kind=getattr(mesh, "kind", "affine"))
    # receive lists: halo elements grouped by owner
    for r in range(world):
        if r == rank:
            continue
        ids = np.flatnonzero(owner[gids[lm.n_own:]] == r) + lm.n_own
        if len(ids):
            lm.recv[r] = ids
    # send lists: owned elements that appear in rank r's halo, increasing global id
    for r in range(world):
        if r == rank:
            continue
        r_owned = owner == r
        # elements of mine adjacent to an element of r
        adj = np.zeros(len(owner), bool)
        nbr_r = nbr_g[r_owned].ravel()
        adj[nbr_r[nbr_r >= 0]] = True
        mine = owned[adj[owned]]
        if len(mine):
            lm.send[r] = g2l[mine]
    return lm


def element_offsets(orders: np.ndarray, ncomp: int = 5) -> np.ndarray:
    n = np.prod(orders.astype(np.int64) + 1, axis=1)
    off = np.zeros(len(orders) + 1, np.int64)
    off[1:] = np.cumsum(ncomp * n)
    return off


def ranges(ids: np.ndarray, off: np.ndarray):
    """Merge the state ranges of element ids (in order) into (start, stop) runs."""
    runs = []
    for e in ids:
        a, b = int(off[e]), int(off[e + 1])
        if runs and runs[-1][1] == a:
            runs[-1][1] = b
        else:
            runs.append([a, b])
    return [tuple(r) for r in runs]


class HaloPlan:
    """State-level exchange plan for the current local orders: per peer rank,
    the (start, stop) ranges of the local state vector to send and to receive
    (ncomp doubles per node: 5 for q, 15 for gradients)."""

    def __init__(self, lm: LocalMesh, local_orders: np.ndarray, ncomp: int = 5):
        off = element_offsets(local_orders, ncomp)
        self.send = {r: ranges(ids, off) for r, ids in lm.send.items()}
        self.recv = {r: ranges(ids, off) for r, ids in lm.recv.items()}
        self.send_len = {r: sum(b - a for a, b in rs) for r, rs in self.send.items()}
        self.recv_len = {r: sum(b - a for a, b in rs) for r, rs in self.recv.items()}
        assert set(self.send) == set(self.recv), "face adjacency is symmetric"


# face f = 2 d + s of an element: tangential directions (a, b) of d
_TAN = ((1, 2), (0, 2), (0, 1))


def face_points(orders_e, f: int) -> int:
    """Nodes of face f of an element of orders (N1, N2, N3)."""
    a, b = _TAN[f >> 1]
    return int((orders_e[a] + 1) * (orders_e[b] + 1))


class TracePlan:
    """Face-trace halo plan (one exchange of partition-boundary
    face traces per residual, two for NS): the face kernels read only the
    nodes of a neighbour element's face toward the owned element, so instead
    of whole element states a rank sends, for every face between one of its
    owned elements A and an element owned by rank r, the trace of A on that
    face (ncomp components x face points, [comp][pt] with pt = ta + n_a tb),
    and receives the traces of r's elements into the same face nodes of its
    halo copies.  Entries are ordered by (global id, face) on both sides, so
    rank r's send list and this rank's receive list from r match one to one.
    Per peer: `send[r]` / `recv[r]` int64 arrays [n][2] = (buffer offset,
    8 local_id + face) for dg_trace_copy, and the buffer lengths."""

    def __init__(self, lm: LocalMesh, local_orders: np.ndarray, ncomp: int = 5):
        orders = np.asarray(local_orders)
        owner_local = np.full(lm.E, lm.rank, np.int64)
        for r, ids in lm.recv.items():
            owner_local[ids] = r
        gids = lm.gids
        owned = np.arange(lm.n_own)
        self.ncomp = ncomp
        self.send, self.recv, self.send_len, self.recv_len = {}, {}, {}, {}
        peers = sorted(set(lm.send) | set(lm.recv))
        for r in peers:
            # send: faces of owned elements whose neighbour is a halo element of rank r
            ent = []
            for e in owned:
                for f in range(6):
                    nb = lm.nbr[e, f]
                    if nb >= lm.n_own and owner_local[nb] == r:
                        ent.append((int(gids[e]), f, int(e)))
            # receive: faces of rank r's halo elements toward an owned element
            rec = []
            for h in range(lm.n_own, lm.E):
                if owner_local[h] != r:
                    continue
                for f in range(6):
                    nb = lm.nbr[h, f]
                    if 0 <= nb < lm.n_own:
                        rec.append((int(gids[h]), f, int(h)))
            self.send[r], self.send_len[r] = self._table(sorted(ent), orders, ncomp)
            self.recv[r], self.recv_len[r] = self._table(sorted(rec), orders, ncomp)

    @staticmethod
    def _table(entries, orders, ncomp):
        t = np.zeros((len(entries), 2), np.int64)
        o = 0
        for i, (_, f, e) in enumerate(entries):
            t[i, 0] = o
            t[i, 1] = 8 * e + f
            o += ncomp * face_points(orders[e], f)
        return t, o


class MigrationPlan:
    """Element moves between two partitions (old_owner -> new_owner) seen from
    `rank`: per peer, the global ids it sends (its old owned elements that the
    peer owns now) and receives (its new owned elements the peer owned),
    increasing global id, with their state lengths (ncomp doubles per node).
    Owned states are kept in increasing global id order on both sides."""

    def __init__(self, old_owner: np.ndarray, new_owner: np.ndarray, orders: np.ndarray, rank: int, world: int,
                 ncomp: int = 5):
        n = ncomp * np.prod(np.asarray(orders, np.int64) + 1, axis=1)
        self.old_ids = np.flatnonzero(old_owner == rank)
        self.new_ids = np.flatnonzero(new_owner == rank)
        self.old_off = np.concatenate([[0], np.cumsum(n[self.old_ids])])
        self.send_ids = [self.old_ids[new_owner[self.old_ids] == r] for r in range(world)]
        self.recv_ids = [self.new_ids[old_owner[self.new_ids] == r] for r in range(world)]
        self.send_len = [int(n[i].sum()) for i in self.send_ids]
        self.recv_len = [int(n[i].sum()) for i in self.recv_ids]
        self.n = n
