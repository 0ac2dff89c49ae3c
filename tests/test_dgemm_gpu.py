"""The FP64 tensor-core GEMM behind every FMM translation (lb_dgemm_cols,
csrc/dgemm_cols.cuh: DMMA 8x8x4 with gathered / permuted columns) against a
plain PyTorch fp64 reference of the same op, on the FMM's shapes (surface m
= 8 / 10 lattices, the Chebyshev grid, rank-sized low-rank factors), odd
strides (8-byte copies) and tails."""

import ctypes

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,K,n,gather,perm,add", [
    (296, 296, 1000, False, False, 0), (488, 488, 777, True, False, 1),
    (729, 729, 300, True, True, 0), (37, 729, 513, True, True, 0),
    (729, 37, 129, False, False, 1), (5, 3, 7, False, False, 0), (64, 488, 1, True, True, 1),
    # one column count per tile of gemm_cols' wave model at the translation
    # shape (dgemm_cols.cuh: 32x32, 64x64, 64x96 with the 4-stage ring,
    # 64x128 with the 3-stage ring, 128x128), gathered and in place
    (488, 488, 740, True, False, 0), (488, 488, 1500, True, False, 1), (488, 488, 3001, True, False, 1),
    (488, 488, 4380, False, False, 0), (488, 488, 8760, True, False, 1), (729, 729, 2200, True, True, 1),
    (296, 296, 6001, True, False, 0)])
def test_dgemm_cols_matches_torch(cuda, M, K, n, gather, perm, add):
    torch = cuda
    from paper_2111_10743_b200 import _lib
    L = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(M * 7 + K)
    A = torch.randn(M, K, dtype=torch.float64, device="cuda", generator=g)
    X = torch.randn(n + 5, K, dtype=torch.float64, device="cuda", generator=g)
    Y0 = torch.randn(n, M, dtype=torch.float64, device="cuda", generator=g)
    Y = Y0.clone()
    cols = torch.randperm(n + 5, device="cuda", generator=g)[:n].to(torch.int64) if gather else None
    tab = torch.stack([torch.randperm(K, device="cuda", generator=g) for _ in range(3)]).to(
        torch.int32) if perm else None
    kp = torch.randint(0, 3, (n + 5,), device="cuda", dtype=torch.int32, generator=g) if perm else None
    _lib.check(L.lb_dgemm_cols(_lib.ptr(A), K, M, K, _lib.ptr(X), K, _lib.ptr(cols), _lib.ptr(tab),
                               _lib.ptr(kp), n, _lib.ptr(Y), M, ctypes.c_double(0.5), add,
                               _lib.stream_handle()))
    Xg = X[cols] if gather else X[:n]
    if perm:
        Xg = torch.gather(Xg, 1, tab[kp[:n].long()].long())  # kp indexed by output column
    ref = 0.5 * (Xg @ A.T) + (Y0 if add else 0)
    assert float((Y - ref).abs().max() / ref.abs().max()) < 1e-14
