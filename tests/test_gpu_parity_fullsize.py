"""BASELINE.json's configurations at FULL length against the f64 oracle (SURVEY.md 8(d) parity
gates): configs[1] exactly (592^3 computed nodes, order 8, 500 steps: 1e-5 after 100 steps,
1e-4 after the run), configs[2]'s gradient at 592^3 over a 64-step window with every 4th
level saved (1e-3, dot test 1e-4), and configs[4] on a reduced grid (order 16, 8 off-node
sources, 1000 steps).  The oracle needs about 4 minutes of a 16-core host for the three
(profiles/r02_parity_fullsize.json holds the figures of the round-2 run); set
SFB_FULLSIZE_STEPS to shorten configs[1] when iterating."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

pytestmark = pytest.mark.gpu


def test_config2_full_length_against_the_oracle():
    import parity_fullsize as pf
    r = pf.config2(int(os.environ.get("SFB_FULLSIZE_STEPS", "500")))
    print(r)
    assert r["traces_absmax"] > 0 and r["wavefield_absmax"] > 0
    assert r["traces_rel_l2_early"] <= 1e-5 and r["wavefield_rel_l2_early"] <= 1e-5
    assert r["traces_rel_l2_full"] <= 1e-4 and r["wavefield_rel_l2_full"] <= 1e-4


def test_config3_gradient_at_full_size_against_the_oracle():
    import parity_fullsize as pf
    r = pf.config3(64)
    print(r)
    assert r["gradient_absmax"] > 0
    assert r["gradient_rel_l2"] <= 1e-3 and r["dot_test_rel"] <= 1e-4
    assert r["traces_rel_l2"] <= 1e-5


def test_config5_reduced_grid_full_length_against_the_oracle():
    import parity_fullsize as pf
    r = pf.config5_reduced(1000)
    print(r)
    assert r["n_src"] == 8 and r["space_order"] == 16 and r["traces_absmax"] > 0
    assert r["traces_rel_l2_early"] <= 1e-5 and r["wavefield_rel_l2_early"] <= 1e-5
    assert r["traces_rel_l2_full"] <= 1e-4 and r["wavefield_rel_l2_full"] <= 1e-4
