"""The oracle at the BENCHMARKED sizes (cfg2 1024^2, cfg4 full, cfg5 at 96^3)
against the reference's own outputs of the same seeded problems
(tests/golden/configs_full.npz, made by the reference): vmult, diagonal and
Newton residual fingerprints bit-equal up to 1e-12 (observed exact)."""
import numpy as np
import pytest

from tests.fullsize import CASES, check_fingerprint, oracle_outputs


@pytest.mark.parametrize("name,levels,tag", CASES)
def test_oracle_full_size_matches_reference(golden, name, levels, tag):
    from paper_1902_08112_b200 import configs
    g = golden["configs_full"]
    prob = configs.make(name, levels)
    chk = g[f"{tag}/checksum"]
    assert np.isclose(prob.state.U.sum(), chk[0], rtol=1e-13, atol=0)
    assert np.isclose(prob.v.sum(), chk[1], rtol=1e-13, atol=0)
    mask = prob.dirichlet.is_constrained | prob.active
    assert mask.sum() == chk[2]
    out = oracle_outputs(prob)
    for key in ("apply", "diagonal", "residual"):
        check_fingerprint(out[key], g, tag, key, 1e-12)
