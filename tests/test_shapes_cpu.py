"""The BASELINE geometry generators (paper_2111_10743_b200/shapes.py) hand
the device geometry build BIT-IDENTICAL chart coefficients to the ones the
reference's own generators pass to build_from_coefficients
(shapes.py:27-45,132-156 + surface.py:310-322; SHA-256 digests from
scripts/make_golden_r2.py geom_coeffs).  No device needed."""

import json
import os

import numpy as np
import pytest

from conftest import GOLD
from treehash import sha


@pytest.fixture(scope="module")
def want():
    with open(os.path.join(GOLD, "geom_coeffs_sha256.json")) as f:
        return json.load(f)


CASES = {
    "icosphere_o5": lambda s: s.icosphere(5, coefficients_only=True),
    "icosphere_o7": lambda s: s.icosphere(7, coefficients_only=True),
    "torus_o7_64x32": lambda s: s.build_torus(7, 64, 32, 2.0, 1.0, coefficients_only=True),
    "torus_o7_12x6": lambda s: s.build_torus(7, 12, 6, 2.0, 1.0, coefficients_only=True),
    "wavy_o9_82x163": lambda s: s.wavy_torus(9, 82, 163, coefficients_only=True),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_chart_coefficients_bit_identical(want, name):
    from paper_2111_10743_b200 import shapes
    cx, cu, cv = CASES[name](shapes)
    assert cx.shape[0] == want[name]["npatches"]
    assert sha(cx, np.float64) == want[name]["x"]
    assert sha(cu, np.float64) == want[name]["dxdu"]
    assert sha(cv, np.float64) == want[name]["dxdv"]


def test_torus_argument_errors():
    from paper_2111_10743_b200 import shapes
    with pytest.raises(ValueError):
        shapes.build_torus(7, 8, 8, 1.0, 2.0)
    with pytest.raises(ValueError):
        shapes.build_torus(7, 3, 8, 2.0, 1.0)
