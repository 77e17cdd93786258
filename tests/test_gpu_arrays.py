"""Host/device plumbing of the numpy-facing twins: the threaded page-locked
staging copies (pffmg_copy_h2d / pffmg_copy_d2h) move exactly the bytes a plain
torch copy moves, for every size class (below one chunk, chunk multiples, more
chunks than ring slots, odd tails) and dtype the twins use."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CH = 4 << 20


@pytest.mark.parametrize("nbytes", [1 << 20, CH - 8, CH, CH + 8, 3 * CH + 4096 + 8, 8 * CH, 11 * CH + 24])
def test_threaded_copies_roundtrip(nbytes, monkeypatch):
    from paper_1902_08112_b200 import arrays
    monkeypatch.setattr(arrays, "THREADED_MIN_H2D", 1 << 20)
    monkeypatch.setattr(arrays, "THREADED_MIN_D2H", 1 << 20)
    rng = np.random.default_rng(nbytes % 1000)
    a = rng.standard_normal(nbytes // 8)
    d = arrays.dev(a)
    assert d.is_cuda and d.dtype == torch.float64
    assert torch.equal(d, torch.from_numpy(a).cuda())
    back = arrays.host(d)
    assert isinstance(back, np.ndarray) and np.array_equal(back, a)
    buf = torch.zeros(a.size, dtype=torch.float64, device="cuda")
    arrays.copy_into(buf, a)
    assert torch.equal(buf, d)


def test_threaded_copies_masks_and_small(monkeypatch):
    from paper_1902_08112_b200 import _lib, arrays
    rng = np.random.default_rng(1)
    m = rng.random(20_000_001) < 0.3
    seen = []
    real = _lib.call
    monkeypatch.setattr(_lib, "call", lambda n_, *a: (seen.append(n_), real(n_, *a))[1])
    d = arrays.dev(m, torch.uint8)
    assert "pffmg_copy_h2d" in seen
    assert torch.equal(d, torch.from_numpy(m.astype(np.uint8)).cuda())
    seen.clear()
    small = rng.standard_normal(1000)
    assert torch.equal(arrays.dev(small), torch.from_numpy(small).cuda()) and not seen   # below THREADED_MIN_H2D
    monkeypatch.setattr(arrays, "THREADED_COPIES", False)
    big = rng.standard_normal(1 << 18)
    assert torch.equal(arrays.dev(big), torch.from_numpy(big).cuda()) and not seen
    assert np.array_equal(arrays.host(arrays.dev(big)), big)
