"""FMM plan structure on the CPU (no device needed): the native octree and
U/V/W/X lists are BIT-EXACT with the reference's _build_tree/_build_lists
(golden arrays from running the reference), and the host-computed unit
operators are bit-identical to the reference's (SHA-256 of the bytes)."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLD, golden


def _h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def sha():
    with open(os.path.join(GOLD, "unit_ops_sha256.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("m", [5, 8, 10])
def test_surface_unit_operators_bit_identical(sha, m):
    from paper_2111_10743_b200.fmm_plan import unit_operators
    o = unit_operators(m, 1)
    p = f"s{m}_"
    assert _h(o["surf"]) == sha[p + "surf"]
    assert _h(o["pinv_up"]) == sha[p + "pinv_up"]
    assert _h(o["pinv_dn"]) == sha[p + "pinv_dn"]
    assert _h(o["m2m"]) == sha[p + "m2m"]
    assert _h(o["l2l"]) == sha[p + "l2l"]
    assert _h(o["canon"]) == sha[p + "canon"]
    assert _h(np.array(o["canon_keys"], dtype=np.int64)) == sha[p + "keys"]
    assert _h(o["off_vec"].astype(np.int64)) == sha[p + "offs"]
    assert _h(o["off_key"].astype(np.int64)) == sha[p + "okey"]
    assert _h(o["off_perm"].astype(np.int64)) == sha[p + "perm"]


@pytest.mark.parametrize("n", [9, 11])
def test_grid_unit_operators_bit_identical(sha, n):
    from paper_2111_10743_b200.fmm_plan import unit_operators_grid
    o = unit_operators_grid(n, 2)
    p = f"g{n}_"
    assert _h(o["pts"]) == sha[p + "pts"]
    assert _h(o["m2m_1d"]) == sha[p + "m2m_1d"]
    assert _h(o["canon"]) == sha[p + "canon"]
    assert _h(np.array(o["canon_keys"], dtype=np.int64)) == sha[p + "keys"]
    assert _h(o["off_vec"].astype(np.int64)) == sha[p + "offs"]
    assert _h(o["off_key"].astype(np.int64)) == sha[p + "okey"]
    assert _h(o["off_perm"].astype(np.int64)) == sha[p + "perm"]
    assert _h(o["vinv"]) == sha[p + "vinv"]


def _csr(lists):
    lens = [0 if x is None else len(x) for x in lists]
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    flat = np.concatenate([np.asarray(x, np.int64) for x in lists if x is not None
                           and len(x)]) if off[-1] else np.zeros(0, np.int64)
    return off, flat


@pytest.mark.parametrize("case", ["u1_", "u2_", "cl_", "cl2_", "sph_"])
def test_tree_and_lists_bit_exact(case):
    from paper_2111_10743_b200.fmm_plan import FmmPlan
    g = golden("fmm_tree.npz")
    buf = int(g[case + "buffer"])
    eps = 1e-6 if buf == 1 else 1e-9
    plan = FmmPlan(g[case + "spos"], g[case + "tpos"], eps, ncrit=int(g[case + "ncrit"]),
                   device_sort=False)
    assert plan.buffer == buf
    t = plan.tree
    assert np.array_equal(t.center, g[case + "center"])
    assert t.half == float(g[case + "half"])
    for name in ("level", "ijk", "parent", "nsrc"):
        assert np.array_equal(getattr(t, name), g[case + name]), name
    assert np.array_equal(t.is_leaf, g[case + "is_leaf"])
    for name, lst in (("children", t.children), ("src_idx", t.src_idx),
                      ("tgt_idx", t.tgt_idx)):
        off, flat = _csr(lst)
        assert np.array_equal(off, g[case + name + "_off"]), name
        assert np.array_equal(flat, g[case + name]), name
    for name, lst in zip(("colleagues", "vlist", "ulist", "wlist", "xlist"), t.lists()):
        off, flat = _csr(lst)
        assert np.array_equal(off, g[case + name + "_off"]), name
        assert np.array_equal(flat, g[case + name]), name  # same order, not just same set


def test_capacity_error_on_pathological_clustering():
    """fmm.py:605-609 (test_fmm.py:135-140)."""
    from paper_2111_10743_b200 import FmmCapacityError
    from paper_2111_10743_b200.fmm_plan import FmmPlan
    pos = np.zeros((200000, 3))
    pos[-1] = [1.0, 0, 0]
    with pytest.raises(FmmCapacityError):
        FmmPlan(pos, np.array([[2.0, 0, 0]]), 1e-6, ncrit=100, device_sort=False)


def test_order_for_eps_thresholds():
    from paper_2111_10743_b200 import order_for_eps
    assert order_for_eps(1e-3) == ("surface", 5, 1)
    assert order_for_eps(1e-6) == ("surface", 8, 1)
    assert order_for_eps(5e-8) == ("surface", 10, 1)
    assert order_for_eps(1e-9) == ("grid", 9, 2)
    assert order_for_eps(1e-10) == ("grid", 11, 2)


def test_lowrank_m2l_factors():
    """fmm_plan.m2l_factors: canon_k ~= A_k B_k within tol * sigma_max per key,
    ranks far below nrep (the reason the low-rank M2L beats the dense
    product), and the packing the C ABI expects (row-major, key order)."""
    from paper_2111_10743_b200.fmm_plan import m2l_factors, m2l_lowrank_tol, unit_operators_grid
    ops = unit_operators_grid(9, 2)
    canon = ops["canon"]
    tol = m2l_lowrank_tol(1e-9)
    assert abs(tol - 1e-11) < 1e-24
    ranks, a, b = m2l_factors(canon, tol)
    nrep = canon.shape[1]
    assert ranks.shape == (canon.shape[0],) and ranks.max() <= 80 and ranks.min() >= 1
    assert a.size == b.size == int(ranks.sum()) * nrep
    off = 0
    for k, r in enumerate(ranks):
        A = a[off * nrep:(off + r) * nrep].reshape(nrep, r)
        B = b[off * nrep:(off + r) * nrep].reshape(r, nrep)
        K = canon[k]
        s0 = np.linalg.norm(K, 2)
        assert np.linalg.norm(K - A @ B, 2) <= 1.01 * tol * s0
        off += r
