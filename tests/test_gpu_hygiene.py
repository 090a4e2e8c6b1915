"""ABI hygiene on the GPU: argument checks of the binding and the
admissibility flag (reading A25) surfaced at synchronising calls."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2210_03523_b200 as m

    m.build()
    return m


def _cube(dg):
    import torch

    mesh = W.cube_mesh(2)
    orders = W.orders_uniform(mesh.E, 3)
    S = dg.Solver(mesh)
    S.set_orders(orders)
    q = torch.from_numpy(W.pulse_state(S.node_coords(), orders, sigma=0.2)).cuda()
    return mesh, orders, S, q


def test_binding_rejects_bad_tensors(dg):
    """The binding checks dtype, device, contiguity and length before a
    pointer reaches the kernels (no out-of-bounds read on a wrong tensor)."""
    import torch

    mesh, orders, S, q = _cube(dg)
    r = torch.empty_like(q)
    S.rhs_eval(q, r)  # the good call works
    with pytest.raises(dg.DGError, match="dtype"):
        S.rhs_eval(q.float(), r)
    with pytest.raises(dg.DGError, match="CUDA"):
        S.rhs_eval(q.cpu(), r)
    with pytest.raises(dg.DGError, match="contiguous"):
        S.rhs_eval(torch.stack([q, q], 1)[:, 0], r)
    with pytest.raises(dg.DGError, match="elements"):
        S.rhs_eval(q[:-1], r)
    with pytest.raises(dg.DGError, match="tau"):
        S.tau_estimate(q, r, tau=torch.empty((mesh.E, 3, 4), dtype=torch.float64, device="cuda"))
    dt = torch.zeros(1, dtype=torch.float64, device="cuda")
    with pytest.raises(dg.DGError, match="dt"):
        S.rk_step(q, r, torch.empty_like(q), dt.float())


@pytest.mark.parametrize("physics", ["euler_affine", "ns_curved"])
def test_admissibility_surfaces(dg, physics):
    """A state with rho < 0 at one node: the residual kernel flags it, the
    next synchronising call (compute_dt with a host value) fails with
    DG_EADMISSIBLE naming the element; the flag is then cleared."""
    import torch

    if physics == "euler_affine":
        mesh, orders, S, q = _cube(dg)
        bad_e = 5
        offq = W.offsets(orders, 5)
    else:
        mesh = W.ogrid_mesh(3, 8, 2, ratio=1.5, g_eta=2)
        orders = W.orders_random(mesh.E, (2, 2, 1), (4, 4, 2), 9)
        nsp = W.ns_params()
        S = dg.Solver(mesh, physics=dg.NS, mu=nsp["mu"], Pr=nsp["Pr"], qinf=nsp["qinf"])
        S.set_orders(orders)
        q = torch.from_numpy(W.freestream_noise_state(orders, (1.0, 1.0, 0.0, 0.0, nsp["p_inf"]), seed=3)).cuda()
        bad_e = 7
        offq = W.offsets(orders, 5)
    qb = q.clone()
    qb[int(offq[bad_e]) + 1] = -0.5  # density of node 1 of element bad_e
    S.rhs_eval(qb)
    with pytest.raises(dg.DGError, match=f"inadmissible.*element {bad_e}"):
        S.compute_dt(q, 0.5, sync=True)
    # cleared: the next synchronising call on a good state succeeds
    S.rhs_eval(q)
    assert S.compute_dt(q, 0.5, sync=True) > 0.0
