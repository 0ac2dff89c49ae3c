"""Hardware probes bench.py states its rooflines from (csrc/probe.cu): they
must compute what they claim to time -- the two-stream row read returns each
row's exact sum, the mixed DMMA / DFMA probe accepts every warp split."""

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nrows,rowlen", [(1, 1), (37, 300), (1000, 2808), (9, 4097)])
def test_read_rows_probe_sums_rows(cuda, nrows, rowlen):
    torch = cuda
    from paper_2111_10743_b200 import _lib
    L = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(nrows * 31 + rowlen)
    # small integers: every partial sum is exact in fp64 whatever the order
    a = torch.randint(-8, 9, (nrows, rowlen), device="cuda", generator=g).double()
    b = torch.randint(-8, 9, (nrows, rowlen), device="cuda", generator=g).double()
    out = torch.full((nrows,), float("nan"), dtype=torch.float64, device="cuda")
    _lib.check(L.lb_probe_read_rows(_lib.ptr(a), _lib.ptr(b), nrows, rowlen, _lib.ptr(out),
                                    _lib.stream_handle()))
    torch.cuda.synchronize()
    assert torch.equal(out, a.sum(1) + b.sum(1))


def test_mixed_pipe_probe_runs_every_split(cuda):
    torch = cuda
    from paper_2111_10743_b200 import _lib
    L = _lib.load()
    scr = torch.zeros(148, dtype=torch.float64, device="cuda")
    for nw in range(0, 9):
        _lib.check(L.lb_probe_mixed(_lib.ptr(scr), 148, 10, 10, nw, _lib.stream_handle()))
    torch.cuda.synchronize()
    assert float(scr.abs().sum()) == 0.0  # the probes never store (their guard value is unreachable)
