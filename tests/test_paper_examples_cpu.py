"""CPU checks of the paper-table driver (paper_2404_10221_b200/paper_examples.py): the golden rows
parse with their citations, and the examples' sources split exactly into e^{-t} A + e^{-2t} B."""
import math

import numpy as np
import pytest

from paper_2404_10221_b200 import inputs as I
from paper_2404_10221_b200 import paper_examples as P


def test_golden_rows_parse_and_cite():
    rows = P.load_rows()
    assert len(rows) == 21 + 21 + 18                     # Tables 1, 2, 3
    for r in rows:
        assert r.table in (1, 2, 3) and len(r.alpha) == r.table and r.source.startswith("P:")
        assert r.M in (1024, 4096, 16384) and r.N1 in (8, 16, 32, 64, 128)
        assert 0 < r.error < 1e-3 and 4.0 < r.it_u < 11.0 and 4.0 < r.it_d < 11.0
    # the Table 1 rows also pinned by the oracle test agree with this file
    t1 = {(r.N1, r.alpha[0]): r for r in rows if r.table == 1 and r.M == 4096}
    assert t1[(16, 1.3)].it_u == 6.6 and t1[(64, 1.9)].error == 8.81e-7


@pytest.mark.parametrize("d", [1, 2, 3])
def test_source_splits_into_two_time_factors(d):
    prob = I.example(d, 7, 16, (1.3, 1.5, 1.7)[:d])
    A, B = P._source_parts(prob)
    for t in (0.1, 0.37, 0.9):
        f = prob.f_closed(t)
        assert np.max(np.abs(f - (math.exp(-t) * A + math.exp(-2 * t) * B))) <= 1e-12 * max(1.0, np.abs(f).max())
