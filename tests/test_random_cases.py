"""Random feature mixes (tests/random_cases.py): every case is valid for the C-ABI host and the oracle
keeps its conservation identities (CPU).  GPU parity on the same cases: tests/test_gpu_random.py."""
import numpy as np
import pytest

import oracle
from paper_2601_03197_b200 import sdas
from random_cases import make_case


@pytest.mark.parametrize("seed", range(0, 40, 3))
def test_random_case_valid_and_conserving(seed):
    p, g, obj = make_case(seed)
    P = sdas.Pipeline(p)
    L = sdas.results_layout(P, sdas.GridView(p, g))
    assert L.n_replicas == len(g["candidates"]) * len(g["arrivals"]) * g["n_seeds"]
    s = oracle.simulate(p, g, records=False, hists=False)["summary"]
    for x in s:
        assert int(x["arrivals"]) == int(x["admitted"]) + int(x["dropped"])
        if x["status"] == 0:                       # finished: every admitted request completed
            assert x["completed"] == x["admitted"]
            assert x["msgs_emitted"] == x["msgs_received"] and x["tokens_emitted"] == x["tokens_received"]
            assert x["completed_int"] <= x["completed"] and x["rejected"] <= x["dropped"]
