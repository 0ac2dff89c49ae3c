"""Sharded device apply (lb_opset_apply_phase + exchanges) emulated in ONE
process on one GPU: every 'rank' is a handle on its own row range, the
exchanges are done by copying rows between the handles' work buffers.  Must
reproduce the unsharded apply (A1/A2/A3, exact and FMM far fields)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _emulate(devs, parts, form, tau, torch):
    n = tau.numel()
    outs = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in devs]
    nph = 3 if form == 3 else 2
    for p in range(nph):
        for d, o in zip(devs, outs):
            d.apply_phase(form, p, tau, o)
        vecs, red = devs[0].phase_exchange(form, p)
        for k in vecs:
            full = torch.zeros(n, dtype=torch.float64, device="cuda")
            for d, (r0, nr) in zip(devs, parts):
                full[r0:r0 + nr] = d.buffers()[0][k][r0:r0 + nr]
            for d in devs:
                d.buffers()[0][k].copy_(full)
        if red:
            s = sum(d.buffers()[1].clone() for d in devs)
            for d in devs:
                d.buffers()[1].copy_(s)
    res = torch.zeros(n, dtype=torch.float64, device="cuda")
    for o, (r0, nr) in zip(outs, parts):
        res[r0:r0 + nr] = o[r0:r0 + nr]
    return res


@pytest.mark.parametrize("fixture,form,far", [
    ("opset_sphere_o3.npz", "a3", "direct"), ("opset_sphere_o3.npz", "a2", "direct"),
    ("opset_sphere_o3.npz", "a1", "direct"), ("opset_torus_o3.npz", "a3", "direct"),
    ("opset_torus_o3.npz", "a3", "fmm")])
def test_emulated_shards_match_unsharded(cuda, fixture, form, far):
    torch = cuda
    from paper_2111_10743_b200 import (CorrectionSet, Geometry, KernelKind,
                                       LayerOperatorSet)
    from paper_2111_10743_b200.fmm_plan import FmmPlan
    from paper_2111_10743_b200.operators import FORMULATIONS, DeviceOperator
    from paper_2111_10743_b200.sharding import partition_rows
    g = golden(fixture)
    geom, cset = Geometry.from_arrays(g), CorrectionSet.from_arrays(g)
    ref_op = LayerOperatorSet(geom, form, 1e-10, corrections=cset, far=far)
    tau = torch.from_numpy(g["tau"]).cuda()
    ref = ref_op.apply(tau)
    nb = geom.nodes_per_patch
    n = geom.nnodes
    code = {"a1": 1, "a2": 2, "a3": 3}[form]
    for world in (2, 3):
        parts = partition_rows(n // nb, nb, world)
        devs, plans = [], []
        for r0, nr in parts:
            d = DeviceOperator(geom, cset, list(FORMULATIONS[form]), row0=r0, nrows=nr)
            if far == "fmm":  # replicated tree, owned target rows (sharding.py)
                pl = FmmPlan(geom.over_nodes, geom.nodes, 1e-10)
                pl.set_target_range(r0, r0 + nr)
                d.set_fmm(pl)
                plans.append(pl)
            devs.append(d)
        ones = torch.ones(n, dtype=torch.float64, device="cuda")
        phi0 = torch.zeros(n, dtype=torch.float64, device="cuda")
        for d, (r0, nr) in zip(devs, parts):
            tmp = torch.zeros(n, dtype=torch.float64, device="cuda")
            d.apply_layer(KernelKind.SINGLE_LAYER, ones, tmp)
            phi0[r0:r0 + nr] = tmp[r0:r0 + nr]
        for d in devs:
            d.set_phi0(phi0)
        if form == "a3" and far == "direct":  # the fused second sweep, as ShardedOperatorSet runs it
            from paper_2111_10743_b200.operators import eta_weights
            phi_eta = torch.from_numpy(eta_weights(geom, cset)).cuda()
            for d in devs:
                d.set_eta_weights(phi_eta)
        got = _emulate(devs, parts, code, tau, torch)
        err = (got - ref).abs().max().item() / ref.abs().max().item()
        # FMM shards share the unsharded tree: the same approximation
        assert err < 1e-12, (world, err)


@pytest.mark.parametrize("far", ["direct", "fmm"])
def test_sharded_set_world1_morton_device_corrections(cuda, far):
    """ShardedOperatorSet's own path on one rank: Morton-permuted patches,
    corrections built on the device for its rows, inputs / outputs in the
    caller's order -- equal to the plain LayerOperatorSet."""
    from paper_2111_10743_b200 import Geometry, LayerOperatorSet
    from paper_2111_10743_b200.sharding import ShardedOperatorSet
    g = golden("opset_torus_o3.npz")
    geom = Geometry.from_arrays(g)
    eps = float(g["eps"])
    ref = LayerOperatorSet(geom, "a3", eps, far=far).apply(g["tau"])
    op = ShardedOperatorSet(geom, "a3", eps, None, far=far)
    got = op.apply(g["tau"])
    assert np.abs(got - ref).max() <= 1e-10 * np.abs(ref).max()


def test_distributed_upward_pass_emulated(cuda):
    """The FMM's upward pass split by source range (lb_fmm_plan_set_source_range)
    with the partial expansions summed by the upward hook: G plans on one GPU,
    each with its rank's sources; pass 1 records every rank's partial
    expansions, pass 2 hands each rank the sum (what the all-reduce does) --
    the result equals the unsplit FMM."""
    torch = cuda
    from paper_2111_10743_b200.fmm_plan import FmmPlan
    rng = np.random.default_rng(5)
    s = rng.standard_normal((40000, 3))
    s /= np.linalg.norm(s, axis=1)[:, None]
    t = s[::3].copy()
    q = torch.from_numpy(rng.standard_normal((2, len(s)))).cuda()
    nt = len(t)

    def run(plan):
        pot = torch.zeros((2, nt), dtype=torch.float64, device="cuda")
        grad = torch.zeros((2, nt, 3), dtype=torch.float64, device="cuda")
        plan.apply_device(q, None, 2, 3, 0, 1, pot, grad)
        torch.cuda.synchronize()
        return pot, grad
    for eps in (1e-6, 1e-9):
        ref = run(FmmPlan(s, t, eps))
        G = 3
        cuts = [0, 13000, 27000, len(s)]
        plans, partial = [], [None] * G
        for r in range(G):
            p = FmmPlan(s, t, eps)
            p.set_source_range(cuts[r], cuts[r + 1])
            plans.append(p)
        for r, p in enumerate(plans):  # pass 1: record the partials
            def rec(up, nd, stream, r=r):
                partial[r] = up.clone()
            p.set_upward_hook(rec)
            run(p)
        total = sum(partial)
        for r, p in enumerate(plans):  # pass 2: the all-reduced expansions
            p.set_upward_hook(lambda up, nd, stream: up.copy_(total))
            pot, grad = run(p)
            assert p._hook_error is None
            # summing the partial expansions in another order moves the result
            # by roundoff, which the surface representation's Tikhonov
            # pseudo-inverse amplifies (measured 4.4e-11 at eps 1e-6; the grid
            # representation stays near 1e-14)
            bar = 1e-9 if eps >= 3e-8 else 1e-11
            for a, b in ((pot, ref[0]), (grad, ref[1])):
                err = (a - b).abs().max().item() / b.abs().max().item()
                assert err < bar, (eps, r, err)
        assert not torch.equal(partial[0], total)  # the split really was partial
