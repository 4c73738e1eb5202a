"""GPU vs oracle, bit-exact, on seeded random feature mixes (tests/random_cases.py): DAGs with fan-out,
routing, tools, KV, classes / priority / admission, guards, pacing, controllers and truncation."""
import pytest

from gpu_parity import full_check
from random_cases import make_case, make_lean_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(120))
def test_random_case_parity(seed):
    p, g, obj = make_case(seed)
    full_check(p, g, objective=obj)


@pytest.mark.parametrize("seed", range(200))
def test_random_lean_case_parity(seed):
    """The same mixes reduced to the LEAN level (one instance per role, a chain of links): its event-skipping
    shortcuts against the oracle on random costs, modes and controllers."""
    p, g, obj = make_lean_case(seed)
    a, _ = full_check(p, g, objective=obj)
    assert a["res"].layout.k1_variant == 2
