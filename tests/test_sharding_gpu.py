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
