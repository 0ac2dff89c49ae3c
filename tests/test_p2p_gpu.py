"""CUDA P2P (csrc/p2p.cu via lb_p2p / lb_p2p_grouped) vs the reference's
golden vectors and vs the C oracle.  Tolerance: fp64 direct sums within 1e-12
relative (max-norm per density normalised by max |ref|, test_fmm.py:41-48)."""

import numpy as np
import pytest

import oracle
from conftest import golden, rel_errs

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _b200():
    import paper_2111_10743_b200 as b
    return b


def test_golden_cloud_all_levels(cuda):
    b = _b200()
    g = golden("p2p_direct.npz")
    res = b.evaluate_direct(b.FmmSources(g["a_src"], g["a_ch"], g["a_dip"]),
                            g["a_tgt"], ("pot", "grad", "hess"))
    assert rel_errs(res.pot, g["a_pot"], 2) < TOL
    assert rel_errs(res.grad, g["a_grad"], 2) < TOL
    assert rel_errs(res.hess, g["a_hess"], 2) < TOL
    # sources == targets (self pairs skipped), charge+dipole on one density
    res = b.evaluate_direct(b.FmmSources(g["b_x"], g["b_ch"], g["b_dip"]),
                            g["b_x"], ("pot", "grad", "hess"))
    assert rel_errs(res.pot, g["b_pot"], 3) < TOL
    assert rel_errs(res.grad, g["b_grad"], 3) < TOL
    assert rel_errs(res.hess, g["b_hess"], 3) < TOL
    h = res.hess
    assert np.array_equal(h, np.swapaxes(h, -1, -2))


def test_config1_direct(cuda):
    """BASELINE config 1: icosphere N=4800, charges w*sigma, pot+grad."""
    b = _b200()
    g = golden("config1.npz")
    q = (g["weights"] * g["sigma"])[None]
    res = b.evaluate_direct(b.FmmSources(g["nodes"], q), g["nodes"],
                            ("pot", "grad"))
    assert rel_errs(res.pot, g["pot"], 1) < TOL
    assert rel_errs(res.grad, g["grad"], 1) < TOL
    assert res.hess is None


def test_known_answers(cuda):
    b = _b200()
    res = b.evaluate_direct(b.FmmSources(np.zeros((1, 3)), np.ones((1, 1))),
                            np.array([[1.0, 0, 0]]), ("pot", "grad"))
    assert res.pot[0, 0] == pytest.approx(1.0, rel=1e-15)
    assert res.grad[0, 0] == pytest.approx([-1.0, 0, 0], rel=1e-15)
    dip = np.zeros((1, 1, 3))
    dip[0, 0] = [0, 0, 1.0]
    res = b.evaluate_direct(b.FmmSources(np.zeros((1, 3)), dipoles=dip),
                            np.array([[0.0, 0, 2.0]]), ("pot",))
    assert res.pot[0, 0] == pytest.approx(0.25, rel=1e-15)
    pos = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    res = b.evaluate_direct(b.FmmSources(pos, np.ones((1, 2))), pos, ("pot",))
    assert res.pot[0, 0] == pytest.approx(1.0, rel=1e-15)


def test_zero_density_stays_zero(cuda):
    b = _b200()
    rng = np.random.default_rng(0)
    pos = rng.uniform(-1, 1, (50, 3))
    ch = rng.standard_normal((3, 50))
    ch[1] = 0.0
    res = b.evaluate_direct(b.FmmSources(pos, ch), rng.uniform(2, 3, (20, 3)),
                            ("pot",))
    assert np.all(res.pot[1] == 0.0)
    assert np.abs(res.pot[0]).max() > 0


@pytest.mark.parametrize("level", [0, 1, 2])
def test_grouped_matches_reference(cuda, level):
    b = _b200()
    g = golden("p2p_direct.npz")
    want = [{"pot"}, {"pot", "grad"}, {"pot", "grad", "hess"}][level]
    out = b.run_grouped_direct(g["c_t_xyz"], g["c_t_out"], g["c_t_off"],
                               g["c_s_xyz"], g["c_s_c"], g["c_s_v"],
                               g["c_s_off"], g["c_use_c"], g["c_use_d"], want,
                               2, 400)
    for k in want:
        ref = g[f"c{level}_{k}"]
        assert np.abs(out[k] - ref).max() <= TOL * np.abs(ref).max(), k


@pytest.mark.parametrize("nt,ns,nd", [(37, 5000, 5), (3000, 129, 1),
                                      (1, 1, 1), (2000, 2000, 2)])
def test_vs_oracle_shapes_and_chunks(cuda, nt, ns, nd):
    """Ragged sizes, density chunking (nd=5 -> 4+1), source splitting."""
    b = _b200()
    rng = np.random.default_rng(nt + ns + nd)
    src = rng.uniform(-1, 1, (ns, 3))
    tgt = np.vstack([rng.uniform(-1, 1, (nt - 1, 3)), src[:1]]) if nt > 1 \
        else src[:1].copy()
    ch = rng.standard_normal((nd, ns))
    dip = rng.standard_normal((nd, ns, 3))
    if nd > 1:
        ch[nd - 1] = 0.0
        dip[0] = 0.0
    res = b.evaluate_direct(b.FmmSources(src, ch, dip), tgt,
                            ("pot", "grad", "hess"))
    pot, grad, hess = oracle.p2p(tgt, src, ch, dip, level=2)
    assert rel_errs(res.pot, pot, nd) < TOL
    assert rel_errs(res.grad, grad, nd) < TOL
    assert rel_errs(res.hess, hess, nd) < TOL


def test_empty_inputs(cuda):
    b = _b200()
    res = b.evaluate_direct(b.FmmSources(np.zeros((0, 3)), np.zeros((2, 0))),
                            np.ones((4, 3)), ("pot", "grad"))
    assert res.pot.shape == (2, 4) and np.all(res.pot == 0)
    assert np.all(res.grad == 0)
    res = b.evaluate_direct(b.FmmSources(np.ones((3, 3)), np.ones((1, 3))),
                            np.zeros((0, 3)), ("pot",))
    assert res.pot.shape == (1, 0)


def test_torch_in_torch_out(cuda):
    b = _b200()
    torch = cuda
    rng = np.random.default_rng(3)
    x = torch.from_numpy(rng.standard_normal((500, 3))).cuda()
    q = torch.from_numpy(rng.standard_normal((1, 500))).cuda()
    res = b.evaluate_direct(b.FmmSources(x, q), x, ("pot", "grad"))
    assert isinstance(res.pot, torch.Tensor) and res.pot.is_cuda
    pot, grad, _ = oracle.p2p(x.cpu().numpy(), x.cpu().numpy(),
                              q.cpu().numpy(), level=1)
    assert rel_errs(res.pot.cpu().numpy(), pot, 1) < TOL


def test_large_sphere_sampled(cuda):
    """N=2e5 sources == targets on the sphere; 256 sampled targets checked
    against the oracle (size-independent spot check at bench scale)."""
    b = _b200()
    rng = np.random.default_rng(105)
    n = 200_000
    x = rng.standard_normal((n, 3))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    q = rng.standard_normal((1, n))
    res = b.evaluate_direct(b.FmmSources(x, q), x, ("pot", "grad"))
    idx = rng.choice(n, 256, replace=False)
    pot, grad, _ = oracle.p2p(x[idx], x, q, level=1)
    assert rel_errs(res.pot[:, idx], pot, 1) < TOL
    assert rel_errs(res.grad[:, idx], grad, 1) < TOL


def test_shape_errors(cuda):
    b = _b200()
    with pytest.raises(ValueError):
        b.FmmSources(np.zeros((3, 2)), np.zeros((1, 3)))
    with pytest.raises(ValueError):
        b.evaluate_direct(b.FmmSources(np.zeros((3, 3)), np.zeros((1, 3))),
                          np.zeros((3, 3)), ("pot", "laplacian"))


def test_inv_sqrt_domain(cuda):
    """The pairwise 1/r (lb_common.cuh inv_sqrt_skip: MUFU.RSQ64H seed + one
    2nd-order fp64 step) over 2^-63 <= r < 2^64, and the coincident-pair skip
    (r2 == 0 -> exactly 0)."""
    import torch
    from paper_2111_10743_b200 import _lib
    L = _lib.load()
    rng = np.random.default_rng(0)
    x = np.exp2(rng.uniform(-126.0, 127.9, 1 << 18))
    x[:3] = [0.0, 1.0, 4.0]
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    _lib.check(L.lb_probe_rsqrt(_lib.ptr(xd), _lib.ptr(yd), len(x), 1,
                                _lib.stream_handle()))
    y = yd.cpu().numpy()
    ref = 1.0 / np.sqrt(x[1:].astype(np.longdouble))
    rel = np.abs((y[1:] - ref) / ref).astype(float)
    assert rel.max() < 1e-15, rel.max()
    assert y[0] == 0.0
    assert abs(y[1] - 1.0) < 1e-15 and abs(y[2] - 0.5) < 1e-15
