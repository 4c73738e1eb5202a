"""GPU vs oracle, bit-exact, on seeded random feature mixes (tests/random_cases.py): DAGs with fan-out,
routing, tools, KV, classes / priority / admission, guards, pacing, controllers and truncation."""
import pytest

from gpu_parity import full_check
from random_cases import make_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(120))
def test_random_case_parity(seed):
    p, g, obj = make_case(seed)
    full_check(p, g, objective=obj)
