"""Pin the oracle: the C restatement and the compiled reference must both
reproduce the reference test suite's known answers."""
import pytest

import kat
from oracle.oracle import Oracle, RefOracle

BACKENDS = [Oracle] + ([RefOracle] if RefOracle.available() else [])


@pytest.mark.parametrize("B", BACKENDS, ids=lambda b: b.__name__)
@pytest.mark.parametrize("check", kat.ALL, ids=lambda f: f.__name__)
def test_known_answers(B, check):
    check(B)
