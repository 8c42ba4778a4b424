"""The engine's exponential variates (rng.hpp:43: E = -log1p(-u), u = x 2^-53):
the table-driven gap function and the series-based service-key function both
stay within 3 ulp of the exactly rounded value (x87 long double reference)."""
import numpy as np
import pytest

import paper_2412_04504_b200 as bb

pytestmark = pytest.mark.gpu


def keys():
    rng = np.random.default_rng(20241204)
    x = [rng.integers(0, 1 << 53, size=400_000, dtype=np.uint64)]
    # u near 0 (E tiny), near 1 (E ~ 36.7), and y = 2^53 - x on the
    # table's subinterval and binade boundaries
    x.append(np.arange(0, 4096, dtype=np.uint64))
    x.append((1 << 53) - 1 - np.arange(0, 4096, dtype=np.uint64))
    y = []
    for e in range(0, 54):
        for m in (0.6875, 0.75, 1.0, 1.0 - 2**-9, 1.0 + 2**-8, 1.375, 1.5):
            v = int(round(m * 2.0**e))
            for d in (-2, -1, 0, 1, 2):
                if 1 <= v + d <= (1 << 53):
                    y.append(v + d)
    x.append((1 << 53) - np.array(sorted(set(y)), dtype=np.uint64))
    return np.concatenate(x)


def ulps(got, x):
    u = x.astype(np.longdouble) * np.longdouble(2.0) ** -53
    want = -np.log1p(-u)
    spacing = np.spacing(np.abs(want.astype(np.float64)))
    return np.abs(got.astype(np.longdouble) - want) / spacing.astype(np.longdouble)


@pytest.mark.parametrize("table", [True, False])
def test_exponential_variate_accuracy(table):
    x = keys()
    got = bb.exponential_variates(x, table=table)
    err = ulps(got, x)
    assert np.all(np.isfinite(got)) and np.all(got >= 0)
    assert got[x == 0][0] == 0.0
    assert float(err.max()) <= 3.0, (float(err.max()), int(x[np.argmax(err)]))
    assert float(err.mean()) <= 0.75
