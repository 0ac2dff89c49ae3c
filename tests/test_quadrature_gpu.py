"""Device near-correction build (csrc/quad.cu) against the
reference's own near maps and corrections (tests/golden/*.npz and
tests/golden/config2_geom.npz, written by scripts/make_golden.py from lapbel;
the config 2-4 correction rows are pinned in tests/test_configs_gpu.py).

Near maps and CSR patterns are integer work: bit-exact.  Correction values:
the device runs the reference's adaptive subdivision, rules, tolerance and
forcing, but sums in a different order (the reference runs numba fastmath),
so an accept decision whose error sits at the leaf tolerance can flip and
move that pair's integral by about the tolerance (0.1 eps per leaf, times
|vinv| in node-weight units).  Measured worst cases: 7.5e-11 of max|value|
and 1.9e-9 of the row's max at eps 1e-10 (config 2); the bars below are
5 eps and 50 eps."""

import os

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KINDS = ("s", "d", "sprime", "grads1", "grads2", "grads3", "spp_plus_dprime")


def _kind(name):
    from paper_2111_10743_b200.operators import as_kind
    return as_kind(name)


def _case(name):
    return golden(name + ".npz")


@pytest.mark.parametrize("name", ["opset_sphere_o3", "opset_torus_o3", "quad_sphere_o7",
                                  "quad_sphere_o9"])
def test_near_map_bit_exact(cuda, name):
    from paper_2111_10743_b200 import Geometry
    from paper_2111_10743_b200.quadrature import build_near_map
    g = _case(name)
    near = build_near_map(Geometry.from_arrays(g), float(g["near_eta"]))
    assert np.array_equal(near.offsets, g["near_offsets"])
    assert np.array_equal(near.patches, g["near_patches"])
    # the reference's list-of-arrays view: self patch first
    lists = near.near
    assert all(lists[t][0] == g["node_patch"][t] for t in range(len(lists)))


def test_near_map_cap_error(cuda):
    from paper_2111_10743_b200 import Geometry
    from paper_2111_10743_b200.quadrature import NearMapCapError, build_near_map
    g = _case("opset_torus_o3")
    with pytest.raises(NearMapCapError):
        build_near_map(Geometry.from_arrays(g), 2.0, cap=4)
    with pytest.raises(ValueError):
        build_near_map(Geometry.from_arrays(g), 0.0)


@pytest.mark.parametrize("name", ["opset_sphere_o3", "opset_torus_o3", "quad_sphere_o7",
                                  "quad_sphere_o9"])
def test_corrections_match_reference(cuda, name):
    """quad_sphere_o9: reference order 9 (config 4's order), where a CTA holds
    only two leaves' basis tables and a self pair's three Duffy roots are
    evaluated in two batches."""
    from paper_2111_10743_b200 import Geometry
    from paper_2111_10743_b200.quadrature import NearMap, build_correction_set
    g = _case(name)
    geom = Geometry.from_arrays(g)
    near = NearMap(float(g["near_eta"]), 128, g["near_offsets"], g["near_patches"])
    kinds = [k for k in KINDS if "corr_" + k in g]
    eps = float(g["eps"])
    cset, t_q = build_correction_set(geom, near, [_kind(k) for k in kinds], eps)
    ip = cset.indptr.cpu().numpy()
    assert np.array_equal(ip, g["corr_indptr"])
    assert np.array_equal(cset.indices.cpu().numpy(), g["corr_indices"])
    rows = np.repeat(np.arange(len(ip) - 1), np.diff(ip))
    for k in kinds:
        v = cset.values[_kind(k)].cpu().numpy()
        ref = g["corr_" + k]
        diff = np.abs(v - ref)
        assert diff.max() <= 5 * eps * np.abs(ref).max(), k
        rowmax = np.maximum.reduceat(np.abs(ref), ip[:-1])
        assert (diff / rowmax[rows]).max() <= 50 * eps, k


def test_bad_eps_rejected(cuda):
    from paper_2111_10743_b200 import Geometry
    from paper_2111_10743_b200.quadrature import NearMap, build_correction_set
    g = _case("opset_sphere_o3")
    near = NearMap(2.0, 128, g["near_offsets"], g["near_patches"])
    with pytest.raises(ValueError):
        build_correction_set(Geometry.from_arrays(g), near, [_kind("s")], 1e-2)


def test_a1_solve_with_device_corrections(cuda):
    """A1 (S + grad S kinds, principal-value constants on the device) on the
    order-3 cube sphere against the reference's A1 solve and apply."""
    import paper_2111_10743_b200 as b
    g = _case("opset_sphere_o3")
    geom = b.Geometry.from_arrays(g)
    near = b.build_near_map(geom, 2.0)
    op = b.LayerOperatorSet(geom, "a1", float(g["eps"]), near=near, far="direct")
    assert op.corrections_built_on == "device"
    np.testing.assert_allclose(op.apply(g["tau"]), g["a1_apply"],
                               atol=1e-6 * np.abs(g["a1_apply"]).max())
    rep = b.solve_laplace_beltrami(op, g["f"], b.SolveConfig(formulation="a1", eps=1e-6,
                                                             eps_gmres=1e-10, max_iter=60))
    u = np.asarray(rep.u.values)
    assert np.linalg.norm(u - g["a1_u"]) / np.linalg.norm(g["a1_u"]) < 1e-5


def test_config2_solve_with_device_corrections(cuda):
    """BASELINE config 2 end to end on the device: near map + corrections
    (reference: 385 s of CPU) + A3 GMRES solve, against the reference's
    solve with its own corrections."""
    import paper_2111_10743_b200 as b
    from paper_2111_10743_b200.quadrature import build_near_map
    g = _case("config2_geom")
    geom = b.Geometry.from_arrays(g)
    near = build_near_map(geom, 2.0)
    op = b.LayerOperatorSet(geom, "a3", float(g["eps"]), near=near, far="direct")
    assert op.t_q > 0 and op.corrections_built_on == "device"
    rep = b.solve_laplace_beltrami(op, g["f"], b.SolveConfig(formulation="a3", eps=1e-10,
                                                             eps_gmres=1e-10))
    u = np.asarray(rep.u.values)
    ref = g["a3_u"]
    assert np.linalg.norm(u - ref) / np.linalg.norm(ref) < 1e-9
    exact = g["u_exact"]
    err = np.linalg.norm(u - exact) / np.linalg.norm(exact)
    ref_err = np.linalg.norm(ref - exact) / np.linalg.norm(exact)
    assert err < 1.01 * ref_err + 1e-9


def test_correction_cache_roundtrip(cuda, tmp_path):
    """corrcache.py through LayerOperatorSet(correction_cache=...): the first
    construction builds on the device and writes the entry, the second loads
    it (no rebuild) and applies identically."""
    import paper_2111_10743_b200 as b
    g = _case("opset_sphere_o3")
    geom = b.Geometry.from_arrays(g)
    path = str(tmp_path / "sphere.lbcorr")
    op1 = b.LayerOperatorSet(geom, "a3", float(g["eps"]), far="direct",
                             correction_cache=path)
    assert op1.corrections_built_on == "device"
    op2 = b.LayerOperatorSet(geom, "a3", float(g["eps"]), far="direct",
                             correction_cache=path)
    assert op2.corrections_built_on == "cache" and op2.t_q == 0.0
    tau = np.asarray(g["tau"])
    assert np.array_equal(op1.apply(tau), op2.apply(tau))
    # another eps is a key miss: rebuilt, entry overwritten
    op3 = b.LayerOperatorSet(geom, "a3", 1e-8, far="direct", correction_cache=path)
    assert op3.corrections_built_on == "device"
