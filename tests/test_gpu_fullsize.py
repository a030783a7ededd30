"""BASELINE sizes against the oracle: C0 (the reference's CPU-runnable case)
and C1 (the bench workload) at full size, Omega from seed 0, through the
product path (tools/parity_full.py; C2-C4 are run by the same tool and their
results committed under profiles/). Bars: top-k sigma within 1e-10 relative,
||UU^T - U'U'^T||_2 and ||VV^T - V'V'^T||_2 within 1e-8, q passes."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["C0", "C1"])
def test_fullsize_parity(fb, orc, name):
    from parity_full import run
    r = run(name)
    print(r)
    assert r["sigma_rel"] <= 1e-10
    assert r["subspace_U"] <= 1e-8 and r["subspace_V"] <= 1e-8
    assert r["passes_gpu"] == r["q"] == r["passes_oracle"]
