"""CPU checks of the comparison rules themselves (tests/parity.py): the O(n) top-K order used for
large inventories equals the full lexsort's prefix, ties included."""
import numpy as np
import pytest

from tests.parity import topk_order


@pytest.mark.parametrize("n,k,levels", [(5000, 10, 7), (20000, 300, 50), (50000, 1000, 3), (9000, 2000, 100000)])
def test_topk_order_equals_lexsort(n, k, levels):
    rng = np.random.default_rng(n + k)
    r = rng.integers(0, levels, n).astype(np.float64) / 8.0      # many exact ties
    full = np.lexsort((np.arange(n), -r))[:k]
    assert (topk_order(r, k) == full).all()
