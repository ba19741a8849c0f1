"""The oracle's generator restatement (oracle/tdp_oracle_gen.c) is netlist-identical to the reference's
generate_synthetic compiled from its own sources (generator.cpp:60-244) and to the product's
O(N log N) generator up to the 1M-cell bench design.  It is what bench.py's reference arm builds its
input with, so that arm never loads the product library."""
import numpy as np
import pytest

from oracle.oracle import Oracle, RefOracle

ARRAYS = ("cell_w", "cell_h", "cell_delay", "cell_fixed", "pin_cell", "pin_term", "pin_off", "pin_dir", "pin_cap",
          "net_start", "net_pins", "sources", "endpoints", "positions")

needs_ref = pytest.mark.skipif(not RefOracle.available(), reason="oracle/_ref not built")


def same(a, b):
    for k in ARRAYS:
        x, y = getattr(a, k), getattr(b, k)
        assert x.shape == y.shape and np.array_equal(x, y), k
    assert a.core == b.core and a.r_unit == b.r_unit and a.c_unit == b.c_unit


@needs_ref
@pytest.mark.parametrize("seed,cells,kw", [(1, 40, {}), (7, 40, {"fail_frac": 0.3}), (3, 300, {}),
                                           (5, 1000, {"fanout": 3.0}), (2, 2000, {"registers": 50}),
                                           (11, 5, {}), (4, 3000, {"fanout": 1.2}), (9, 600, {"fanout": 6.0})])
def test_oracle_generator_matches_reference(seed, cells, kw):
    same(Oracle.generate(seed=seed, cells=cells, **kw), RefOracle.generate(seed=seed, cells=cells, **kw))


@needs_ref
@pytest.mark.slow
@pytest.mark.parametrize("cells", [10000])
def test_oracle_generator_matches_reference_large(cells):
    same(Oracle.generate(seed=1, cells=cells, fail_frac=0.7), RefOracle.generate(seed=1, cells=cells, fail_frac=0.7))


@pytest.mark.parametrize("seed,cells", [(1, 200000), (1, 1000000)])
def test_oracle_generator_matches_product_at_bench_sizes(seed, cells):
    from paper_2503_11674_b200.engine import generate
    same(Oracle.generate(seed=seed, cells=cells, fail_frac=0.8), generate(seed=seed, cells=cells, fail_frac=0.8,
                                                                          calibrate=False))


def test_oracle_generator_rejects_bad_specs():
    from oracle.oracle import OracleError
    for kw in ({"cells": 0}, {"fanout": 0.0}, {"fail_frac": 1.5}, {"r_unit": 0.0}):
        with pytest.raises(OracleError):
            Oracle.generate(**kw)
