"""On-disk correction cache (paper_2111_10743_b200/corrcache.py, SURVEY
§8(f) #4): byte layout round trip, key invalidation on every field, and the
reference's own corrections (tests/golden/quad_sphere_o7.npz) surviving a
save/load bit for bit.  Host-only: no GPU."""

import os

import numpy as np
import pytest

from conftest import golden
from paper_2111_10743_b200 import CorrectionSet, Geometry, KernelKind
from paper_2111_10743_b200.corrcache import (CacheKeyMismatch, load_corrections,
                                             mesh_hash, save_corrections)


def _golden_set():
    g = golden("quad_sphere_o7.npz")
    return g, Geometry.from_arrays(g), CorrectionSet.from_arrays(g)


def test_roundtrip_reference_corrections(tmp_path):
    g, geom, cs = _golden_set()
    mh = mesh_hash(geom)
    p = os.path.join(tmp_path, "c.lbcorr")
    save_corrections(p, cs, mh, 1e-10, 2.0)
    kinds = list(cs.values)
    back = load_corrections(p, mh, kinds, 1e-10, 2.0)
    assert np.array_equal(back.indptr, cs.indptr)
    assert np.array_equal(back.indices, cs.indices)
    for k in kinds:
        assert np.array_equal(back.values[k], cs.values[k])
    # a subset of the kinds is served from the same entry
    one = load_corrections(p, mh, [KernelKind.SPRIME], 1e-10, 2.0)
    assert list(one.values) == [KernelKind.SPRIME]
    # size = header + codes + arrays, exactly
    n, nnz = len(cs.indptr) - 1, cs.nnz
    nk = len(kinds)
    want = 80 + nk + (-nk % 8) + 8 * (n + 1) + 4 * nnz + (-(4 * nnz) % 8) + 8 * nnz * nk
    assert os.path.getsize(p) == want


def test_key_mismatch_on_every_field(tmp_path):
    g, geom, cs = _golden_set()
    mh = mesh_hash(geom)
    p = os.path.join(tmp_path, "c.lbcorr")
    save_corrections(p, cs, mh, 1e-10, 2.0)
    kinds = list(cs.values)
    moved = Geometry.from_arrays(g)
    moved.nodes = moved.nodes.copy()
    moved.nodes[0, 0] += 1e-15
    for args in ((mesh_hash(moved), kinds, 1e-10, 2.0),
                 (mh, kinds, 1e-9, 2.0),
                 (mh, kinds, 1e-10, 1.5),
                 (mh, [KernelKind.GRAD_S1], 1e-10, 2.0)):
        with pytest.raises(CacheKeyMismatch):
            load_corrections(p, *args)
    with pytest.raises(FileNotFoundError):
        load_corrections(os.path.join(tmp_path, "absent"), mh, kinds, 1e-10, 2.0)
    with open(p, "r+b") as fh:  # truncated entry
        fh.truncate(os.path.getsize(p) - 8)
    with pytest.raises(CacheKeyMismatch):
        load_corrections(p, mh, kinds, 1e-10, 2.0)
