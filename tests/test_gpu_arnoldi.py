"""pffmg_arnoldi_mgs (one Arnoldi step of krylov.py:97-110) against a numpy
restatement of the reference's MGS, on both library paths: the one-launch
cooperative kernel (vectors the size of the BASELINE 2D/3D configs) and the
multi-launch sweep (small vectors).  Covers the plain sweep, the conditional
second sweep (w nearly inside span V) and the w = 0 breakdown."""
import numpy as np
import pytest
import torch

from paper_1902_08112_b200 import _lib

pytestmark = pytest.mark.gpu


def mgs_reference(V, w):
    """krylov.py:97-110: MGS, re-orthogonalise when ||w|| < 1e-3 ||w0||."""
    w = w.copy()
    j = V.shape[0] - 1
    h = np.zeros(j + 2)
    w0 = np.linalg.norm(w)
    for i in range(j + 1):
        h[i] = V[i] @ w
        w -= h[i] * V[i]
    reorth = np.linalg.norm(w) < 1e-3 * w0
    if reorth:
        for i in range(j + 1):
            c = V[i] @ w
            h[i] += c
            w -= c * V[i]
    h[j + 1] = np.linalg.norm(w)
    if h[j + 1] != 0.0:
        w = w / h[j + 1]
    return h, w, reorth


def run_device(V, w, m):
    n = V.shape[1]
    j = V.shape[0] - 1
    Vd = torch.zeros((m + 1, n), dtype=torch.float64, device="cuda")
    Vd[: j + 1] = torch.as_tensor(V, device="cuda")
    Vd[j + 1] = torch.as_tensor(w, device="cuda")
    h = torch.zeros(m + 1, dtype=torch.float64, device="cuda")
    ctl = torch.zeros(3 + 64, dtype=torch.float64, device="cuda")
    _lib.call("pffmg_arnoldi_mgs", _lib.ptr(Vd), Vd.stride(0), j, _lib.ptr(Vd[j + 1]), n, _lib.ptr(h),
              _lib.ptr(ctl), _lib.stream())
    torch.cuda.synchronize()
    return h[: j + 2].cpu().numpy(), Vd[j + 1].cpu().numpy(), bool(ctl[2].item())


def basis(n, k, seed):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, k)))
    return Q.T.copy(), rng


@pytest.mark.parametrize("n", [1000, 3_151_875])          # multi-launch path / one-launch path (cfg2 size)
@pytest.mark.parametrize("j", [0, 5, 12])
def test_arnoldi_step_matches_mgs(n, j):
    V, rng = basis(n, j + 1, 10 + j)
    w = rng.standard_normal(n)
    h_ref, w_ref, re_ref = mgs_reference(V, w)
    h, wd, re = run_device(V, w, 30)
    assert not re and not re_ref
    np.testing.assert_allclose(h, h_ref, rtol=1e-11, atol=1e-12 * np.abs(h_ref).max())
    assert np.linalg.norm(wd - w_ref) <= 1e-11 * np.linalg.norm(w_ref)


@pytest.mark.parametrize("n", [1000, 3_151_875])
def test_arnoldi_second_sweep(n):
    j = 4
    V, rng = basis(n, j + 1, 3)
    span = V.T @ rng.standard_normal(j + 1)
    noise = rng.standard_normal(n)
    w = span + 1e-5 * np.linalg.norm(span) / np.linalg.norm(noise) * noise   # almost inside span V
    h_ref, w_ref, re_ref = mgs_reference(V, w)
    h, wd, re = run_device(V, w, 30)
    assert re_ref and re
    np.testing.assert_allclose(h[: j + 1], h_ref[: j + 1], rtol=1e-9, atol=1e-12 * np.abs(h_ref).max())
    assert abs(h[j + 1] - h_ref[j + 1]) <= 1e-6 * h_ref[j + 1]
    # the re-orthogonalised direction is orthogonal to the basis to rounding
    assert np.abs(V @ wd).max() <= 1e-10


@pytest.mark.parametrize("n", [1000, 3_151_875])
def test_arnoldi_breakdown_keeps_w(n):
    j = 2
    V, _ = basis(n, j + 1, 5)
    w = np.zeros(n)
    h, wd, _ = run_device(V, w, 30)
    assert h[j + 1] == 0.0
    assert not wd.any()
