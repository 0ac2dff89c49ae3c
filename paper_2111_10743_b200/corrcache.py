"""On-disk cache of near corrections (the reference's
SPEC.md:268 asks for it, its package does not implement it).

A cache entry holds one CorrectionSet (the shared CSR pattern plus one value
array per kind, quadrature.py:691-700) keyed by (mesh hash, kinds, eps, eta).
A lookup whose key differs in ANY field is a miss (the entry is rebuilt and
overwritten), so a cache can never serve corrections of another geometry or
tolerance.

Binary layout (little endian, version 1), documented here and in DESIGN.md:

    offset  size        field
    0       8           magic b"LBCORR\\x00\\x01"
    8       32          mesh hash: SHA-256 over the geometry arrays (below)
    40      8  f64      eps
    48      8  f64      eta
    56      8  u64      n      (rows = columns = nodes)
    64      8  u64      nnz
    72      4  u32      nkinds
    76      4  u32      reserved (0)
    80      nkinds      kind codes (u8, KIND_CODE order of operators.py)
    ...     pad to a multiple of 8
            8 (n+1)     indptr  int64
            4 nnz       indices int32, padded to a multiple of 8 bytes
            8 nnz       values of kind 0, kind 1, ... (f64), in header order

The mesh hash covers order, nodes, normals, weights, over_nodes,
over_weights, node_patch and the chart coefficients when present: everything
the correction build reads.  Host IO only (numpy); device-resident sets are
copied to the host to be written and loaded back as host arrays.
"""

from __future__ import annotations

import hashlib
import os
import struct

import numpy as np

from .operators import KIND_CODE, CorrectionSet, KernelKind, as_kind

__all__ = ["mesh_hash", "save_corrections", "load_corrections",
           "cached_correction_set", "CacheKeyMismatch"]

MAGIC = b"LBCORR\x00\x01"
_HDR = struct.Struct("<8s32sddQQII")
_CODE_KIND = {v: k for k, v in KIND_CODE.items()}


class CacheKeyMismatch(LookupError):
    """The file exists but was written for another (mesh, kinds, eps, eta)."""


def mesh_hash(disc) -> bytes:
    h = hashlib.sha256()
    h.update(str(int(disc.order)).encode())
    for name in ("nodes", "normals", "weights", "over_nodes", "over_weights",
                 "node_patch", "coeffs_x", "coeffs_dxdu", "coeffs_dxdv"):
        a = getattr(disc, name, None)
        if a is None:
            continue
        a = np.ascontiguousarray(a)
        h.update(name.encode())
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.digest()


def _host(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


def save_corrections(path, cset: CorrectionSet, mhash: bytes, eps: float, eta: float):
    """Write `cset` (every kind it holds) under the key (mhash, kinds, eps, eta)."""
    kinds = list(cset.values)
    indptr = np.ascontiguousarray(_host(cset.indptr), dtype="<i8")
    indices = np.ascontiguousarray(_host(cset.indices), dtype="<i4")
    n, nnz = len(indptr) - 1, len(indices)
    tmp = f"{path}.tmp{os.getpid()}"
    with open(tmp, "wb") as fh:
        fh.write(_HDR.pack(MAGIC, mhash, float(eps), float(eta), n, nnz, len(kinds), 0))
        codes = bytes(KIND_CODE[k] for k in kinds)
        fh.write(codes + b"\x00" * (-len(codes) % 8))
        fh.write(indptr.tobytes())
        fh.write(indices.tobytes())
        fh.write(b"\x00" * (-(4 * nnz) % 8))
        for k in kinds:
            fh.write(np.ascontiguousarray(_host(cset.values[k]), dtype="<f8").tobytes())
    os.replace(tmp, path)  # readers never see a half-written entry


def load_corrections(path, mhash: bytes, kinds, eps: float, eta: float) -> CorrectionSet:
    """Load the entry at `path`; raises FileNotFoundError when absent and
    CacheKeyMismatch when its key differs (any field) or a kind is missing."""
    want = [as_kind(k) for k in kinds]
    with open(path, "rb") as fh:
        raw = fh.read(_HDR.size)
        if len(raw) < _HDR.size:
            raise CacheKeyMismatch(f"{path}: truncated header")
        magic, h, e, et, n, nnz, nk, _ = _HDR.unpack(raw)
        if magic != MAGIC:
            raise CacheKeyMismatch(f"{path}: not a correction cache (version 1)")
        codes = fh.read(nk)
        if len(codes) < nk or any(c not in _CODE_KIND for c in codes):
            raise CacheKeyMismatch(f"{path}: truncated or unknown kind codes")
        have = [_CODE_KIND[c] for c in codes]
        if h != mhash or e != float(eps) or et != float(eta) or \
                any(k not in have for k in want):
            raise CacheKeyMismatch(f"{path}: key (mesh, kinds, eps, eta) differs")
    base = _HDR.size + nk + (-nk % 8)
    size = base + 8 * (n + 1) + 4 * nnz + (-(4 * nnz) % 8) + 8 * nnz * nk
    if os.path.getsize(path) != size:
        raise CacheKeyMismatch(f"{path}: size {os.path.getsize(path)} != {size} "
                               "from the header")
    mm = np.memmap(path, mode="r", dtype=np.uint8)
    off = base
    indptr = np.frombuffer(mm, dtype="<i8", count=n + 1, offset=off)
    off += 8 * (n + 1)
    indices = np.frombuffer(mm, dtype="<i4", count=nnz, offset=off)
    off += 4 * nnz + (-(4 * nnz) % 8)
    vals = {}
    for k in have:
        if k in want:
            vals[k] = np.array(np.frombuffer(mm, dtype="<f8", count=nnz, offset=off))
        off += 8 * nnz
    return CorrectionSet(np.array(indptr), np.array(indices), vals, (n, n))


def cached_correction_set(path, disc, near, kinds, eps: float, eta: float = 2.0):
    """CorrectionSet for (disc, kinds, eps, eta): from `path` on a key match,
    else built on the device (quadrature.build_correction_set) and written to
    `path`.  Returns (cset, t_q seconds, hit)."""
    from .quadrature import build_correction_set
    mh = mesh_hash(disc)
    # the pattern comes from `near`, so the key carries the near map's own eta
    # (a map built with another tolerance must never hit this entry)
    eta = float(getattr(near, "eta", eta))
    try:
        return load_corrections(path, mh, kinds, eps, eta), 0.0, True
    except (FileNotFoundError, CacheKeyMismatch):
        pass
    cset, t_q = build_correction_set(disc, near, kinds, eps)
    save_corrections(path, cset, mh, eps, eta)
    return cset, t_q, False


# keep the kind table closed over the enum (a new kind needs a new code)
assert set(_CODE_KIND.values()) <= set(KernelKind)
