"""FmmPlan / evaluate_fmm / order_for_eps: drop-in for the FMM half of
lapbel.fmm (`fmm.py:225-1011`).

The plan (octree, U/V/W/X lists, bit-exact with `_build_tree`/`_build_lists`)
is built natively in libb200lb (`lb_fmm_plan_create`: device Morton keys +
radix sort, host DFS numbering and list walks); `apply` runs every pass on the
B200 (`lb_fmm_apply`).  The unit-box translation operators are plan-time
constants computed here on the host with numpy/LAPACK, restating
`_unit_operators` (fmm.py:287-354) and `_unit_operators_grid`
(fmm.py:431-481) operation for operation, so the device FMM evaluates the SAME
approximation as the reference (not only one within eps of the truth).
"""

from __future__ import annotations

import ctypes
from functools import lru_cache
from itertools import permutations, product

import numpy as np

from . import _lib

__all__ = ["order_for_eps", "unit_operators", "unit_operators_grid",
           "expansion_grid", "FmmPlan", "evaluate_fmm", "TreeView"]

UE_SCALE, UC_SCALE, DC_SCALE, DE_SCALE = 1.05, 2.85, 1.05, 2.85  # fmm.py:228-231
TIK_ALPHA = 1e-9                                                  # fmm.py:232


def order_for_eps(eps: float):
    """(representation, size, separation buffer) for a requested tolerance
    (fmm.py:357-382, same thresholds)."""
    if eps >= 1e-3:
        return "surface", 5, 1
    if eps >= 1e-4:
        return "surface", 6, 1
    if eps >= 1e-5:
        return "surface", 7, 1
    if eps >= 1e-6:
        return "surface", 8, 1
    if eps >= 2e-7:
        return "surface", 9, 1
    if eps >= 3e-8:
        return "surface", 10, 1
    if eps >= 1e-9:
        return "grid", 9, 2
    return "grid", 11, 2


def m2l_slices_for(eps: float, nrep: int) -> int:
    """Int8 slice count of the tensor-core M2L for a tolerance (B200 design
    choice, no reference counterpart).  With S slices of 7 bits the FMM
    result moves from the fp64-M2L result by about 2^(-7S) / 4 relative
    (measured: S=4 2.8e-10, S=5 7e-12 (grid) .. 4e-11 (surface), S=6 6e-14,
    scripts/m2l_probe.py); S is the smallest count with 2^(-7S) <= eps / 128,
    i.e. a deviation near eps / 500, and at most 8 (fp64 roundoff).  0 (fp64
    DGEMM) when the expansion is too large for the kernel (nrep > 2048)."""
    if nrep > 2048:
        return 0
    s = int(np.ceil((np.log2(1.0 / eps) + 7.0) / 7.0))
    return int(min(8, max(3, s)))


_LOWRANK_CACHE: dict = {}


def _lowrank(K: np.ndarray, tol: float, rng) -> tuple:
    """Truncated factorization K ~= A B keeping the singular values above
    tol * sigma_max: a randomized range finder (Gaussian sketch of width k,
    doubled until the sketch's last singular value drops below the
    tolerance) followed by an exact SVD of the k x n projection, so a
    1331 x 1331 operator of rank ~100 costs O(n^2 k) instead of O(n^3)."""
    n = K.shape[1]
    k = min(n, 96)
    while True:
        Q, _ = np.linalg.qr(K @ rng.standard_normal((n, k)))
        ub, sv, vt = np.linalg.svd(Q.T @ K, full_matrices=False)
        if k >= n or sv[-1] <= 0.01 * tol * sv[0]:
            break
        k = min(n, 2 * k)
    r = max(1, int((sv > tol * sv[0]).sum()))
    return np.ascontiguousarray((Q @ ub[:, :r]) * sv[:r]), np.ascontiguousarray(vt[:r]), r


def m2l_factors(canon: np.ndarray, tol: float):
    """Truncated SVD of every canonical M2L matrix (B200 design option, no
    reference counterpart): canon_k ~= A_k B_k keeping the singular values
    above tol * sigma_max(canon_k), so the M2L of one column costs
    2 nrep r_k instead of nrep^2 (the grid operators at n = 9 have r_k <= 63,
    mean 36, at tol 1e-11).  Returns (ranks int32, A packed, B packed)."""
    key = (id(canon), canon.shape, float(tol))
    if key in _LOWRANK_CACHE:
        return _LOWRANK_CACHE[key]
    rng = np.random.default_rng(20211110)  # deterministic sketches
    ranks, As, Bs = [], [], []
    for K in canon:
        a, b, r = _lowrank(K, tol, rng)
        ranks.append(r)
        As.append(a)
        Bs.append(b)
    out = (np.asarray(ranks, dtype=np.int32), np.concatenate([a.ravel() for a in As]),
           np.concatenate([b.ravel() for b in Bs]))
    _LOWRANK_CACHE[key] = out
    return out


def m2l_lowrank_tol(eps: float) -> float:
    """SVD truncation of the low-rank M2L: eps / 100 (the M2L then moves the
    FMM result by far less than its requested precision), in [1e-13, 1e-8]."""
    return float(min(1e-8, max(1e-13, eps / 100.0)))


# ---------------------------------------------------------------------------
# unit-box operators (host precompute, cached like the reference's lru_cache)


def expansion_grid(m: int) -> np.ndarray:
    """Cube-surface lattice of the m x m x m grid on [-1, 1]^3, lexicographic
    (i, j, k) order (fmm.py:243-253)."""
    g = np.array([(i, j, k) for i in range(m) for j in range(m)
                  for k in range(m)
                  if min(i, j, k) == 0 or max(i, j, k) == m - 1], dtype=float)
    return 2.0 * g / (m - 1) - 1.0


def _inv_dist(tpts, spts):
    """1/|t - s| (fmm.py:256-258)."""
    diff = tpts[:, None, :] - spts[None, :, :]
    return 1.0 / np.sqrt(np.einsum("tsk,tsk->ts", diff, diff))


def _tikhonov_pinv(a):
    """Tikhonov-damped pseudo-inverse, alpha = 1e-9 sigma_max (fmm.py:237-240)."""
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    filt = s / (s * s + (TIK_ALPHA * s[0]) ** 2)
    return (vt.T * filt) @ u.T


def _cube_symmetries():
    """The 48 signed permutation matrices (fmm.py:269-279 order)."""
    out = []
    for p in permutations(range(3)):
        for sg in product((1.0, -1.0), repeat=3):
            mat = np.zeros((3, 3))
            for r in range(3):
                mat[r, p[r]] = sg[r]
            out.append(mat)
    return out


def _lattice_map(labels, mat):
    """p with mat @ labels[i] == labels[p[i]] (fmm.py:261-266)."""
    where = {tuple(q): i for i, q in enumerate(labels)}
    moved = labels @ mat.T.astype(np.int64)
    return np.array([where[tuple(q)] for q in moved], dtype=np.int64)


def _offset_tables(labels, buffer, kernel):
    """Canonical M2L matrices (a <= b <= c, c > buffer, insertion order of
    fmm.py:321-327 / 450-456) and, for every lattice offset d outside the
    near field, (canonical index, point permutation) (fmm.py:329-347)."""
    dmax = 2 * buffer + 1
    keys = [(a, b, c) for a in range(dmax + 1) for b in range(a, dmax + 1)
            for c in range(b, dmax + 1) if c > buffer]
    canon = [kernel(np.array(k, float)) for k in keys]
    kidx = {k: i for i, k in enumerate(keys)}
    mats = _cube_symmetries()
    offs, okey, operm = [], [], []
    rng = range(-dmax, dmax + 1)
    for d in product(rng, rng, rng):
        if max(abs(x) for x in d) <= buffer:
            continue
        ck = tuple(sorted(abs(int(x)) for x in d))
        for mat in mats:
            if tuple((mat @ np.array(d, float)).round().astype(int)) == ck:
                offs.append(d)
                okey.append(kidx[ck])
                operm.append(_lattice_map(labels, mat.round().astype(np.int64)))
                break
        else:  # pragma: no cover - the cube group always maps d
            raise AssertionError("no cube symmetry maps the offset")
    return (keys, np.array(canon), np.array(offs, dtype=np.int32),
            np.array(okey, dtype=np.int32), np.array(operm, dtype=np.int32))


@lru_cache(maxsize=8)
def unit_operators(m: int, buffer: int = 1) -> dict:
    """Equivalent-surface operators for lattice size m (fmm.py:287-354)."""
    surf = expansion_grid(m)
    ue, uc, dc, de = (surf * UE_SCALE, surf * UC_SCALE, surf * DC_SCALE,
                      surf * DE_SCALE)
    pinv_up = _tikhonov_pinv(_inv_dist(uc, ue))
    pinv_dn = _tikhonov_pinv(_inv_dist(dc, de))
    octs = np.array([[i, j, k] for i in (-1, 1) for j in (-1, 1)
                     for k in (-1, 1)], dtype=float)
    m2m = np.array([pinv_up @ _inv_dist(uc, 0.5 * ue + 0.5 * o) for o in octs])
    l2l = np.array([_inv_dist(dc, 2.0 * de - o) for o in octs])
    labels = np.round((surf + 1.0) * (m - 1) / 2.0).astype(np.int64) * 2 - (m - 1)
    keys, canon, offs, okey, operm = _offset_tables(
        labels, buffer, lambda k: _inv_dist(dc, ue + 2.0 * k))
    return {"rep": "surface", "m": m, "surf": surf, "pts": surf,
            "pinv_up": pinv_up, "pinv_dn": pinv_dn, "m2m": m2m, "l2l": l2l,
            "canon_keys": keys, "canon": canon, "off_vec": offs,
            "off_key": okey, "off_perm": operm}


def cheb_nodes(n):
    """Chebyshev points of the first kind (fmm.py:389-390)."""
    return np.cos(np.pi * (2.0 * np.arange(n) + 1.0) / (2.0 * n))


def _cheb_values(n, x):
    """T_0..T_{n-1} at x and first/second derivatives (fmm.py:393-410)."""
    x = np.asarray(x, dtype=float)
    t = np.empty((x.size, n))
    dt = np.empty((x.size, n))
    d2t = np.empty((x.size, n))
    t[:, 0], dt[:, 0], d2t[:, 0] = 1.0, 0.0, 0.0
    if n > 1:
        t[:, 1], dt[:, 1], d2t[:, 1] = x, 1.0, 0.0
    for k in range(2, n):
        t[:, k] = 2.0 * x * t[:, k - 1] - t[:, k - 2]
        dt[:, k] = 2.0 * t[:, k - 1] + 2.0 * x * dt[:, k - 1] - dt[:, k - 2]
        d2t[:, k] = 4.0 * dt[:, k - 1] + 2.0 * x * d2t[:, k - 1] - d2t[:, k - 2]
    return t, dt, d2t


@lru_cache(maxsize=8)
def cheb_vinv(n):
    return np.linalg.inv(_cheb_values(n, cheb_nodes(n))[0])


def lagrange_basis(n, x):
    """Lagrange basis at the Chebyshev nodes evaluated at x (fmm.py:419-428)."""
    return _cheb_values(n, x)[0] @ cheb_vinv(n)


@lru_cache(maxsize=8)
def unit_operators_grid(n: int, buffer: int) -> dict:
    """Chebyshev-grid operators (fmm.py:431-481)."""
    x1 = cheb_nodes(n)
    gx, gy, gz = np.meshgrid(x1, x1, x1, indexing="ij")
    pts = np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])
    m2m_1d = np.array([lagrange_basis(n, 0.5 * x1 + 0.5 * s)
                       for s in (-1.0, 1.0)])
    lab1 = 2 * np.arange(n) - (n - 1)
    lx, ly, lz = np.meshgrid(lab1, lab1, lab1, indexing="ij")
    labels = np.column_stack([lx.ravel(), ly.ravel(), lz.ravel()])
    keys, canon, offs, okey, operm = _offset_tables(
        labels, buffer, lambda k: _inv_dist(pts, pts + 2.0 * k))
    return {"rep": "grid", "n": n, "m": n, "x1": x1, "pts": pts,
            "m2m_1d": m2m_1d, "vinv": cheb_vinv(n), "canon_keys": keys,
            "canon": canon, "off_vec": offs, "off_key": okey,
            "off_perm": operm}


# ---------------------------------------------------------------------------
# the plan


class _OpsStruct(ctypes.Structure):
    _fields_ = [("rep", ctypes.c_int), ("m", ctypes.c_int), ("nrep", ctypes.c_int),
                ("pts", ctypes.c_void_p), ("pinv_up", ctypes.c_void_p),
                ("pinv_dn", ctypes.c_void_p), ("m2m", ctypes.c_void_p),
                ("l2l", ctypes.c_void_p), ("ncanon", ctypes.c_int),
                ("canon", ctypes.c_void_p), ("noff", ctypes.c_int),
                ("off_vec", ctypes.c_void_p), ("off_key", ctypes.c_void_p),
                ("off_perm", ctypes.c_void_p), ("vinv", ctypes.c_void_p)]


_TREE_CODES = {name: i for i, name in enumerate((
    "level", "ijk", "parent", "is_leaf", "nsrc", "children_off", "children",
    "src_sorted", "tgt_sorted", "src_lo", "src_hi", "tgt_lo", "tgt_hi",
    "colleagues_off", "colleagues", "v_off", "v", "u_off", "u", "w_off", "w",
    "x_off", "x"))}

_bound = False


def _bind():
    global _bound
    L = _lib.load()
    if not _bound:
        P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.lb_fmm_plan_create.argtypes = [P, I64, P, I64, I32, I32, I32,
                                         ctypes.POINTER(P)]
        L.lb_fmm_plan_destroy.argtypes = [P]
        L.lb_fmm_plan_info.argtypes = [P, P, P]
        L.lb_fmm_plan_export.argtypes = [P, I32, P]
        L.lb_fmm_plan_set_operators.argtypes = [P, ctypes.POINTER(_OpsStruct)]
        L.lb_fmm_apply.argtypes = [P, P, P, I32, ctypes.c_uint32,
                                   ctypes.c_uint32, I32, P, P, P, P]
        L.lb_fmm_plan_set_timing.argtypes = [P, I32]
        L.lb_fmm_plan_set_m2l_factors.argtypes = [P, P, P, P]
        L.lb_fmm_plan_set_target_range.argtypes = [P, I64, I64]
        L.lb_fmm_plan_set_source_range.argtypes = [P, I64, I64]
        L.lb_fmm_plan_set_upward_hook.argtypes = [P, P, P]
        L.lb_fmm_stage_times.argtypes = [P, P]
        L.lb_fmm_setup_times.argtypes = [P, P]
        _bound = True
    return L


class TreeView:
    """The reference's `_Tree` fields (fmm.py:542-556) read back from the
    native plan: level, ijk, parent, children, is_leaf, src_idx, tgt_idx,
    nsrc, levels, centers, halves, center, half."""

    def __init__(self, plan):
        L = _bind()
        sizes = np.zeros(10, dtype=np.int64)
        geom = np.zeros(4)
        _lib.check(L.lb_fmm_plan_info(plan, sizes.ctypes.data_as(ctypes.c_void_p),
                                      geom.ctypes.data_as(ctypes.c_void_p)))
        self.sizes = sizes
        nbox, nlev, ns, nt = (int(x) for x in sizes[:4])
        lens = {"level": nbox, "ijk": 3 * nbox, "parent": nbox,
                "is_leaf": nbox, "nsrc": nbox, "children_off": nbox + 1,
                "children": int(sizes[4]), "src_sorted": ns,
                "tgt_sorted": nt, "src_lo": nbox, "src_hi": nbox,
                "tgt_lo": nbox, "tgt_hi": nbox, "colleagues_off": nbox + 1,
                "colleagues": int(sizes[5]), "v_off": nbox + 1, "v": int(sizes[6]),
                "u_off": nbox + 1, "u": int(sizes[7]), "w_off": nbox + 1,
                "w": int(sizes[8]), "x_off": nbox + 1, "x": int(sizes[9])}
        raw = {}
        for name, n in lens.items():
            a = np.zeros(max(n, 1), dtype=np.int64)
            _lib.check(L.lb_fmm_plan_export(plan, _TREE_CODES[name],
                                            a.ctypes.data_as(ctypes.c_void_p)))
            raw[name] = a[:n]
        self.raw = raw
        self.center = geom[:3].copy()
        self.half = float(geom[3])
        self.level = raw["level"]
        self.ijk = raw["ijk"].reshape(nbox, 3)
        self.parent = raw["parent"]
        self.is_leaf = raw["is_leaf"].astype(bool)
        self.nsrc = raw["nsrc"]
        self.children = self._split("children")
        ss, ts = raw["src_sorted"], raw["tgt_sorted"]
        self.src_idx = [ss[raw["src_lo"][b]:raw["src_hi"][b]] if self.is_leaf[b]
                        else None for b in range(nbox)]
        self.tgt_idx = [ts[raw["tgt_lo"][b]:raw["tgt_hi"][b]] if self.is_leaf[b]
                        else None for b in range(nbox)]
        self.levels = [np.where(self.level == li)[0] for li in range(nlev)]
        self.halves = self.half / (2.0 ** self.level)
        self.centers = (self.center - self.half) + (self.ijk + 0.5) * \
            (2.0 * self.halves)[:, None]

    def _split(self, name):
        off, flat = self.raw[name + "_off"], self.raw[name]
        return [flat[off[b]:off[b + 1]] for b in range(len(off) - 1)]

    def lists(self):
        """colleagues, vlist, ulist, wlist, xlist as per-box arrays."""
        return tuple(self._split(k) for k in ("colleagues", "v", "u", "w", "x"))


class FmmPlan:
    """Reusable geometry plan: octree, interaction lists, unit operators
    (fmm.py:722-782), resident on the B200."""

    def __init__(self, source_positions, target_positions, eps,
                 ncrit: int = 120, m: int | None = None,
                 buffer: int | None = None, rep: str | None = None,
                 device_sort: bool | None = None, m2l="auto", xw: str = "lists"):
        self.spos = np.ascontiguousarray(_host(source_positions), dtype=float)
        self.tpos = np.ascontiguousarray(_host(target_positions), dtype=float)
        self.eps = float(eps)
        rep_auto, m_auto, buf_auto = order_for_eps(self.eps)
        self.rep = rep if rep is not None else rep_auto
        self.m = m if m is not None else m_auto
        self.buffer = buffer if buffer is not None else buf_auto
        self.ncrit = int(ncrit)
        L = _bind()
        if device_sort is None:
            device_sort = _lib.torch().cuda.is_available()
        h = ctypes.c_void_p()
        _lib.check(L.lb_fmm_plan_create(
            self.spos.ctypes.data_as(ctypes.c_void_p), self.spos.shape[0],
            self.tpos.ctypes.data_as(ctypes.c_void_p), self.tpos.shape[0],
            self.ncrit, self.buffer, 1 if device_sort else 0, ctypes.byref(h)),
            "lb_fmm_plan_create")
        self._h = h
        self._L = L
        if self.rep == "surface":
            self.ops = unit_operators(self.m, self.buffer)
            self.nrep = self.ops["pts"].shape[0]
        else:
            self.ops = unit_operators_grid(self.m, self.buffer)
            self.nrep = self.m ** 3
        self._set_operators()
        self._tree = None
        self.set_m2l(m2l)
        self.xw = "lists"
        self.set_xw(xw)

    def set_xw(self, xw: str = "lists"):
        """How X- and W-list entries are evaluated (the lists themselves are
        always the reference's, fmm.py:650-715).  "lists": as the reference
        does (sources on check points, fmm.py:888-911; equivalent charges on
        targets, fmm.py:966-988).  "direct": an X entry of a target LEAF with
        2.5 nt <= nrep and a W entry whose box is a leaf with <= nrep sources
        are summed directly, leaf sources on leaf targets (lb_fmm_plan_set_xw):
        exact where the reference approximates, and fewer pair evaluations on
        surfaces (BASELINE config 3: 757 M X-list lattice pairs -> 116 M
        direct pairs per density).  No reference counterpart; results move
        within eps."""
        if xw not in ("lists", "direct"):
            raise ValueError(f"xw must be 'lists' or 'direct', not {xw!r}")
        _lib.check(self._L.lb_fmm_plan_set_xw(self._h, 1 if xw == "direct" else 0),
                   "lb_fmm_plan_set_xw")
        self.xw = xw

    def set_m2l(self, m2l="auto"):
        """M2L arithmetic: "fp64" (DGEMM on the dense canonical matrices, the
        reference's arithmetic), "auto" = "lowrank" (truncated-SVD factors at
        m2l_lowrank_tol(eps), two thin fp64 DGEMMs: the canonical M2L
        matrices have rank <= 63 of 729 at 1e-11, so this beats the dense
        tensor-core product), or an explicit tcgen05 int8 slice count in
        [3, 8] (m2l_slices_for(eps) sizes it; 8 = fp64 roundoff)."""
        if m2l == "fp64":
            s = 0
        elif m2l in ("auto", "lowrank"):
            ranks, a, b = m2l_factors(self.ops["canon"], m2l_lowrank_tol(self.eps))
            _lib.check(self._L.lb_fmm_plan_set_m2l_factors(
                self._h, ranks.ctypes.data_as(ctypes.c_void_p), a.ctypes.data_as(ctypes.c_void_p),
                b.ctypes.data_as(ctypes.c_void_p)), "lb_fmm_plan_set_m2l_factors")
            self.m2l_ranks = ranks
            s = -1
        else:
            s = int(m2l)
        _lib.check(self._L.lb_fmm_plan_set_m2l(self._h, s), "lb_fmm_plan_set_m2l")
        self.m2l_slices = s

    def _set_operators(self):
        o = self.ops
        keep = []

        def p(a, dt=np.float64):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a.ctypes.data_as(ctypes.c_void_p)
        s = _OpsStruct()
        s.rep = 0 if self.rep == "surface" else 1
        s.m = self.m
        s.nrep = self.nrep
        s.pts = p(o["pts"])
        if self.rep == "surface":
            s.pinv_up, s.pinv_dn = p(o["pinv_up"]), p(o["pinv_dn"])
            s.m2m, s.l2l = p(o["m2m"]), p(o["l2l"])
        else:
            s.m2m, s.vinv = p(o["m2m_1d"]), p(o["vinv"])
        s.ncanon = len(o["canon_keys"])
        s.canon = p(o["canon"])
        s.noff = o["off_vec"].shape[0]
        s.off_vec = p(o["off_vec"], np.int32)
        s.off_key = p(o["off_key"], np.int32)
        s.off_perm = p(o["off_perm"], np.int32)
        _lib.check(self._L.lb_fmm_plan_set_operators(self._h, ctypes.byref(s)),
                   "lb_fmm_plan_set_operators")

    # reference-compatible views of the plan structure
    @property
    def tree(self) -> TreeView:
        if self._tree is None:
            self._tree = TreeView(self._h)
        return self._tree

    @property
    def colleagues(self):
        return self.tree.lists()[0]

    @property
    def vlist(self):
        return self.tree.lists()[1]

    @property
    def ulist(self):
        return self.tree.lists()[2]

    @property
    def wlist(self):
        return self.tree.lists()[3]

    @property
    def xlist(self):
        return self.tree.lists()[4]

    def set_timing(self, on=True):
        _lib.check(self._L.lb_fmm_plan_set_timing(self._h, 1 if on else 0))

    def set_target_range(self, t0: int = 0, t1: int = -1):
        """Owned targets [t0, t1) (lb_fmm_plan_set_target_range; t1 < 0: all).
        The tree and lists stay the reference's; only the owned targets'
        outputs are computed (a sharded apply's rows)."""
        _lib.check(self._L.lb_fmm_plan_set_target_range(self._h, int(t0), int(t1)),
                   "lb_fmm_plan_set_target_range")

    def set_source_range(self, s0: int = 0, s1: int = -1):
        """Owned sources [s0, s1) of the upward pass (lb_fmm_plan_set_source_range;
        s1 < 0: all): P2M + M2M cover only these, and the upward hook must sum
        the ranks' partial expansions (a sharded apply)."""
        _lib.check(self._L.lb_fmm_plan_set_source_range(self._h, int(s0), int(s1)),
                   "lb_fmm_plan_set_source_range")

    def set_upward_hook(self, fn):
        """fn(up, nd, stream): called on the apply's stream between the M2M and
        the M2L with the (nbox, nd, nrep) upward expansions as a CUDA tensor
        view (lb_fmm_plan_set_upward_hook); None removes it."""
        self._hook_fn = fn  # kept so a caller can swap the hook and put it back
        if fn is None:
            self._hook = None
            _lib.check(self._L.lb_fmm_plan_set_upward_hook(self._h, None, None))
            return
        t = _lib.torch()

        def _cb(user, up, count, nd, stream):
            try:
                view = _device_array(up, count, t)
                fn(view, int(nd), stream)
            except Exception as exc:  # noqa: BLE001 - never unwind through C
                self._hook_error = exc
        self._hook_error = None
        self._hook = _HOOK_T(_cb)
        _lib.check(self._L.lb_fmm_plan_set_upward_hook(
            self._h, ctypes.cast(self._hook, ctypes.c_void_p), None))

    def stage_times(self):
        """Device ms of gather+P2M, M2M, M2L, X, L2L, L2T, leaf, scatter, total."""
        ms = np.zeros(9)
        _lib.check(self._L.lb_fmm_stage_times(self._h, ms.ctypes.data_as(ctypes.c_void_p)))
        return dict(zip(("p2m", "m2m", "m2l", "x", "l2l", "l2t", "leaf",
                         "scatter", "total"), ms.tolist()))

    def setup_times(self):
        """Host ms of the plan setup: keys+sort, tree, lists, device state
        (first apply), total."""
        ms = np.zeros(5)
        _lib.check(self._L.lb_fmm_setup_times(self._h, ms.ctypes.data_as(ctypes.c_void_p)))
        return dict(zip(("sort", "tree", "lists", "device", "total"), ms.tolist()))

    def work_counts(self):
        """Algorithmic work of one apply per density, from the tree and lists
        (fmm.py:823-988): pairwise-kernel pair counts of the stages that run
        the 1/r kernel (P2M lattice, X list, leaf U / own-DE / W parts) and
        the M2L's V pairs with its flops (low-rank: 4 nrep r_k per pair,
        dense: 2 nrep^2).  Targets outside an owned range are not excluded."""
        t = self.tree
        r = t.raw
        leaf = t.is_leaf
        ns_box = np.where(leaf, r["src_hi"] - r["src_lo"], 0)
        nt_box = np.where(leaf, r["tgt_hi"] - r["tgt_lo"], 0)
        nrep = self.nrep

        def per_box_sum(off, idx, w):
            v = np.zeros(len(off) - 1)
            if len(idx):
                s = np.concatenate([[0.0], np.cumsum(w[idx], dtype=np.float64)])
                v = s[off[1:]] - s[off[:-1]]
            return v
        nsf = ns_box.astype(float)
        u_src = per_box_sum(r["u_off"], r["u"], nsf)
        x_src = per_box_sum(r["x_off"], r["x"], nsf)
        w_cnt = np.diff(r["w_off"]).astype(float)
        if self.xw == "direct":  # the moves lb_fmm_plan_set_xw makes (fmm_apply.cu build_device)
            xd = leaf & (nt_box > 0) & (5 * nt_box <= 2 * nrep)
            u_src = u_src + np.where(xd, x_src, 0.0)
            x_src = np.where(xd, 0.0, x_src)
            wd_box = leaf & (ns_box <= nrep)          # W members evaluated directly
            w_dir_src = per_box_sum(r["w_off"], r["w"], np.where(wd_box, nsf, 0.0))
            w_dir_cnt = per_box_sum(r["w_off"], r["w"], wd_box.astype(float))
            u_src = u_src + w_dir_src
            w_cnt = w_cnt - w_dir_cnt
        surface = self.rep == "surface"
        out = {"u_pairs": float(np.dot(nt_box, u_src)),
               "w_pairs": float(np.dot(nt_box, w_cnt)) * nrep,
               "de_pairs": float(nt_box.sum()) * nrep if surface else 0.0,
               "x_pairs": float(x_src.sum()) * nrep,
               "p2m_pairs": float(ns_box.sum()) * nrep if surface else 0.0,
               "v_pairs": float(len(r["v"])), "nrep": nrep}
        if self.m2l_slices < 0:  # low-rank: V pairs per canonical key x 4 nrep r_k
            okey = self.ops["off_key"]
            cnt = self._v_pairs_per_key(okey)
            out["m2l_flops"] = float(np.dot(cnt, 4.0 * nrep * self.m2l_ranks))
        else:
            out["m2l_flops"] = out["v_pairs"] * 2.0 * nrep * nrep
        return out

    def _v_pairs_per_key(self, okey):
        """V pairs per canonical key: offset = ijk(src) - ijk(tgt) at one level."""
        t = self.tree
        r = t.raw
        tgt = np.repeat(np.arange(len(r["v_off"]) - 1), np.diff(r["v_off"]))
        d = t.ijk[r["v"]] - t.ijk[tgt]
        ov = self.ops["off_vec"]
        base = int(np.abs(ov).max()) + 1
        code = lambda a: ((a[:, 0] + base) * (2 * base + 1) + (a[:, 1] + base)) \
            * (2 * base + 1) + (a[:, 2] + base)  # noqa: E731
        lut = dict(zip(code(ov).tolist(), okey.tolist()))
        keys = np.array([lut[c] for c in code(d).tolist()], dtype=np.int64)
        return np.bincount(keys, minlength=len(self.ops["canon_keys"])).astype(float)

    def apply_device(self, charges, dipoles, nd, cmask, dmask, level, pot,
                     grad=None, hess=None, stream=None):
        _lib.check(self._L.lb_fmm_apply(
            self._h, _lib.ptr(charges), _lib.ptr(dipoles), nd, cmask, dmask,
            level, _lib.ptr(pot), _lib.ptr(grad), _lib.ptr(hess),
            _lib.stream_handle(stream)), "lb_fmm_apply")

    def apply(self, charges, dipoles, outputs=("pot",), c_active=None,
              d_active=None):
        """fmm.py:784-990."""
        from .fmm import _alloc_device_result, _finish, _level, _parse_outputs
        want = _parse_outputs(outputs)
        host = not (_lib.is_torch(charges) or _lib.is_torch(dipoles))
        if charges is not None and charges.ndim == 1:
            charges = charges[None]
        if dipoles is not None and dipoles.ndim == 2:
            dipoles = dipoles[None]
        nd = charges.shape[0] if charges is not None else dipoles.shape[0]
        if c_active is None:
            c_active = np.ones(nd, bool) if charges is not None else np.zeros(nd, bool)
        if d_active is None:
            d_active = np.ones(nd, bool) if dipoles is not None else np.zeros(nd, bool)
        cm = _lib.mask_of(c_active) if charges is not None else 0
        dm = _lib.mask_of(d_active) if dipoles is not None else 0
        ch = _lib.to_device(charges) if cm else None
        dp = _lib.to_device(dipoles) if dm else None
        level = _level(want)
        pot, grad, hess = _alloc_device_result(nd, self.tpos.shape[0], level)
        if self.tpos.shape[0] == 0:
            return _finish(want, pot, grad, hess, host)
        if cm | dm == 0:
            pot.zero_()
            if grad is not None:
                grad.zero_()
            if hess is not None:
                hess.zero_()
        else:
            self.apply_device(ch, dp, nd, cm, dm, level, pot, grad, hess)
        return _finish(want, pot, grad, hess, host)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._L.lb_fmm_plan_destroy(h)
            except Exception:  # pragma: no cover
                pass
            self._h = None


_HOOK_T = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                           ctypes.c_int, ctypes.c_void_p)


class _CudaArray:
    """A __cuda_array_interface__ over a raw device pointer (zero copy)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None, "stream": None}


def _device_array(ptr, n, t):
    return t.as_tensor(_CudaArray(ptr, n), device="cuda")


def _host(a):
    if _lib.is_torch(a):
        return a.detach().cpu().numpy()
    return a


def evaluate_fmm(sources, targets, eps, outputs=("pot",), ncrit: int = 120,
                 m2l="auto"):
    """FMM evaluation matching evaluate_direct to relative tolerance eps
    (fmm.py:993-1011): eps in [1e-12, 1e-3] else ValueError; all-zero input
    returns zeros without building a plan."""
    from .fmm import _alloc_device_result, _finish, _level, _parse_outputs
    if not (1e-12 <= eps <= 1e-3):
        raise ValueError(f"eps {eps} outside [1e-12, 1e-3]")
    if not (sources.charge_active.any() or sources.dipole_active.any()):
        want = _parse_outputs(outputs)
        host = not _lib.is_torch(targets)
        nt = targets.shape[0]
        pot, grad, hess = _alloc_device_result(sources.nd, nt, _level(want))
        for x in (pot, grad, hess):
            if x is not None:
                x.zero_()
        return _finish(want, pot, grad, hess, host)
    plan = FmmPlan(sources.positions, targets, eps, ncrit=ncrit, m2l=m2l)
    res = plan.apply(sources.charges, sources.dipoles, outputs,
                     sources.charge_active, sources.dipole_active)
    if _lib.is_torch(targets) and not _lib.is_torch(res.pot):
        t = _lib.torch()
        res = type(res)(*(None if x is None else t.from_numpy(x).cuda()
                          for x in (res.pot, res.grad, res.hess)))
    return res
