"""Generator identity at the larger spec sizes: the product's O(N log N) generator and
the oracle's restatement are netlist-identical to the reference's generate_synthetic, compiled from its own
sources, at 40K and 100K cells (the reference's int slot expression stays in range up to ~1.4e5 cells;
above that only product == oracle is checked, tests/test_oracle_gen.py).  Host-only; ~1.5 min."""
import numpy as np
import pytest

from oracle.oracle import Oracle, RefOracle
from paper_2503_11674_b200.engine import generate

pytestmark = [pytest.mark.slow, pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")]

ARRAYS = ("cell_w", "cell_h", "cell_delay", "cell_fixed", "pin_cell", "pin_term", "pin_off", "pin_dir", "pin_cap",
          "net_start", "net_pins", "sources", "endpoints", "positions")


@pytest.mark.parametrize("cells", [40000, 100000])
def test_generators_identical_to_reference(cells):
    ref = RefOracle.generate(seed=1, cells=cells, fail_frac=0.7)
    for ours in (generate(seed=1, cells=cells, fail_frac=0.7, calibrate=False),
                 Oracle.generate(seed=1, cells=cells, fail_frac=0.7)):
        for k in ARRAYS:
            a, b = getattr(ours, k), getattr(ref, k)
            assert a.shape == b.shape and np.array_equal(a, b), (cells, k)
        assert ours.core == ref.core and ours.r_unit == ref.r_unit and ours.c_unit == ref.c_unit
