"""The fast generator is netlist-identical to the reference's generate_synthetic
(same mt19937_64 stream): every array except the calibrated clock is compared
bitwise against the reference compiled from its own sources.  Host logic only
(calibrate=False), so this runs without a GPU."""
import re

import numpy as np
import pytest

from oracle.oracle import RefOracle
from paper_2503_11674_b200.engine import generate

pytestmark = pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")

ARRAYS = ("cell_w", "cell_h", "cell_delay", "cell_fixed", "pin_cell", "pin_term", "pin_off", "pin_dir", "pin_cap",
          "net_start", "net_pins", "sources", "endpoints", "positions")


@pytest.mark.parametrize("seed,cells,kw", [(1, 40, {}), (7, 40, {"fail_frac": 0.3}), (3, 300, {}),
                                           (5, 1000, {"fanout": 3.0}), (2, 2000, {"registers": 50}),
                                           (11, 5, {}), (4, 3000, {"fanout": 1.2})])
def test_netlist_identical_to_reference(seed, cells, kw):
    ref = RefOracle.generate(seed=seed, cells=cells, **kw)
    ours = generate(seed=seed, cells=cells, calibrate=False, **kw)
    for k in ARRAYS:
        a, b = getattr(ours, k), getattr(ref, k)
        assert a.shape == b.shape and np.array_equal(a, b), k
    assert ours.core == ref.core and ours.r_unit == ref.r_unit and ours.c_unit == ref.c_unit


@pytest.mark.slow
def test_netlist_identical_10k():
    ref = RefOracle.generate(seed=1, cells=10000, fail_frac=0.7)
    ours = generate(seed=1, cells=10000, fail_frac=0.7, calibrate=False)
    for k in ARRAYS:
        assert np.array_equal(getattr(ours, k), getattr(ref, k)), k


def test_generator_errors_match_reference():
    from paper_2503_11674_b200.engine import ValidationError
    for kw, msg in [({"cells": 0}, "n_cells must be >= 1"), ({"fanout": 0.0}, "avg_fanout must be > 0"),
                    ({"fail_frac": 1.5}, "target_fail_fraction must be in [0, 1]")]:
        with pytest.raises(ValidationError, match=re.escape(msg)):
            generate(calibrate=False, **kw)
