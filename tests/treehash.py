"""SHA-256 digests of an FmmPlan's octree and interaction lists in the
canonical layout scripts/make_golden_r2.py hashes the reference's
_build_tree/_build_lists output with (fmm.py:559-715): per-box arrays as
int64 (is_leaf as bool, center as fp64), per-box lists as CSR (int64
offsets + int64 flat values, leaves' src_idx/tgt_idx, empty for non-leaves)."""

import hashlib

import numpy as np


def sha(a, dtype):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=dtype)).tobytes()).hexdigest()


def _leaf_csr(sorted_idx, lo, hi, is_leaf):
    lens = np.where(is_leaf, hi - lo, 0).astype(np.int64)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    parts = [sorted_idx[a:b] for a, b, l in zip(lo, hi, is_leaf) if l and b > a]
    flat = np.concatenate(parts).astype(np.int64) if parts else np.zeros(0, np.int64)
    return off, flat


def digests(tv):
    """tv: paper_2111_10743_b200.fmm_plan.TreeView."""
    r = tv.raw
    out = {"nbox": int(len(tv.level)), "nleaf": int(np.sum(tv.is_leaf)),
           "center": sha(tv.center, np.float64), "half": float(tv.half),
           "level": sha(tv.level, np.int64), "ijk": sha(tv.ijk, np.int64),
           "parent": sha(tv.parent, np.int64), "nsrc": sha(tv.nsrc, np.int64),
           "is_leaf": sha(tv.is_leaf, np.bool_)}
    lists = {"children": (r["children_off"], r["children"]),
             "src_idx": _leaf_csr(r["src_sorted"], r["src_lo"], r["src_hi"], tv.is_leaf),
             "tgt_idx": _leaf_csr(r["tgt_sorted"], r["tgt_lo"], r["tgt_hi"], tv.is_leaf),
             "colleagues": (r["colleagues_off"], r["colleagues"]),
             "vlist": (r["v_off"], r["v"]), "ulist": (r["u_off"], r["u"]),
             "wlist": (r["w_off"], r["w"]), "xlist": (r["x_off"], r["x"])}
    for nm, (off, flat) in lists.items():
        out[nm + "_off"] = sha(off, np.int64)
        out[nm] = sha(flat, np.int64)
        out[nm + "_len"] = int(off[-1])
    return out


def compare(got, want):
    """Names of the fields whose digest (or size) differs."""
    keys = [k for k in want if k not in ("ncrit", "buffer", "t_tree_s", "t_lists_s")]
    return [k for k in keys if got.get(k) != want[k]]
