"""BASELINE config 5 at full size (10^6 sources = targets on the unit
sphere, seed 105): the native host octree + lists (csrc/fmm_tree.cpp, the
cross-check the device build is compared with) are BIT-EXACT against the
reference's _build_tree/_build_lists (fmm.py:559-715), checked through
SHA-256 digests of every array (tests/golden/config5_tree_sha256.json,
scripts/make_golden_r2.py config5_tree: 71,922 boxes, 6.99 M V-list
entries at buffer 2).  The device build is checked against the same digests
in tests/test_config5_gpu.py."""

import json
import os

import pytest

from conftest import GOLD
from treehash import compare, digests


@pytest.fixture(scope="module")
def want():
    with open(os.path.join(GOLD, "config5_tree_sha256.json")) as f:
        return json.load(f)


def test_cloud_is_the_reference_cloud(want):
    from paper_2111_10743_b200.shapes import sphere_cloud
    from treehash import sha
    import numpy as np
    assert sha(sphere_cloud(want["n"], want["seed"]), np.float64) == want["x_sha"]


@pytest.mark.parametrize("buffer,eps", [(1, 1e-6), (2, 1e-9)])
def test_host_tree_and_lists_bit_exact_at_1e6(want, buffer, eps):
    from paper_2111_10743_b200.fmm_plan import FmmPlan
    from paper_2111_10743_b200.shapes import sphere_cloud
    x = sphere_cloud(want["n"], want["seed"])
    plan = FmmPlan(x, x, eps, ncrit=120, device_sort=False)
    assert plan.buffer == buffer
    bad = compare(digests(plan.tree), want[f"b{buffer}"])
    assert not bad, bad
