"""The EXACT K1 pivot shortcut (dbag_exact.cu pivot_order_fast / pivot_verified)
against the selection loop it replaces: Eigen's unblocked LDLT pivot search as
restated in oracle.cpp ldlt_solve (first maximum of the remaining |diagonal|,
then a transposition). The shortcut sorts 32-bit keys with a 25-comparator
network and is accepted only when verify() holds; whenever it is accepted its
order must be the selection loop's, bit for bit."""
import struct

import numpy as np

NET = [(0, 1), (3, 4), (6, 7), (1, 2), (4, 5), (7, 8), (0, 1), (3, 4), (6, 7), (0, 3),
       (3, 6), (0, 3), (1, 4), (4, 7), (1, 4), (2, 5), (5, 8), (2, 5), (1, 3), (5, 7),
       (2, 6), (4, 6), (2, 4), (2, 3), (5, 6)]


def selection_order(a):
    a, o = list(a), list(range(9))
    for k in range(9):
        big, best = k, a[k]
        for i in range(k + 1, 9):
            if a[i] > best:
                best, big = a[i], i
        a[k], a[big] = a[big], a[k]
        o[k], o[big] = o[big], o[k]
    return o


def hi_word(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0] >> 32


def fast_order(a):
    key = [(hi_word(a[i]) & 0x7FFFFFF0) | (15 - i) for i in range(9)]
    for i, j in NET:
        key[i], key[j] = max(key[i], key[j]), min(key[i], key[j])
    o = [15 - (k & 15) for k in key]
    d = [a[x] for x in o]
    ok = all(d[p] > d[p + 1] or (p < 7 and d[p] == d[p + 1] and o[p] == 6 and o[p + 1] == 7)
             for p in range(8))
    return o if ok else None


def test_network_sorts_by_zero_one_principle():
    assert len(NET) == 25
    for bits in range(1 << 9):
        a = [(bits >> i) & 1 for i in range(9)]
        for i, j in NET:
            a[i], a[j] = max(a[i], a[j]), min(a[i], a[j])
        assert all(a[k] >= a[k + 1] for k in range(8))


def test_shortcut_equals_selection_loop_when_accepted():
    rng = np.random.default_rng(0)
    accepted = 0
    for t in range(60000):
        mode = t % 6
        if mode == 0:    # distinct, wide dynamic range
            a = rng.standard_normal(9) * 10.0 ** rng.uniform(-3, 6, 9)
        elif mode == 1:  # many ties: fall back
            a = rng.integers(0, 4, 9).astype(float)
        elif mode == 2:  # the structural H66 == H77 tie
            a = rng.uniform(1, 2, 9)
            a[7] = a[6]
        elif mode == 3:  # equal high words, different low words
            a = rng.uniform(1, 2) * (1 + rng.integers(-3, 3, 9) * 2.0 ** -45)
        elif mode == 4:  # the tie with every other value larger (7 first)
            a = rng.uniform(1.0, 2.0, 9)
            a[7] = a[6]
            for i in range(6):
                a[i] = a[6] * rng.uniform(1.01, 2)
            a[8] = a[6] * rng.uniform(1.01, 2)
        else:            # NaN / inf with the tie
            a = rng.uniform(0, 2, 9)
            a[rng.integers(9)] = np.nan if rng.random() < 0.5 else np.inf
            a[7] = a[6]
        a = [abs(float(x)) for x in a]
        f = fast_order(a)
        if f is not None:
            accepted += 1
            assert f == selection_order(a), (a, f)
    assert accepted > 20000


def selection_order_n(a):
    a, o = list(a), list(range(len(a)))
    n = len(a)
    for k in range(n):
        big, best = k, a[k]
        for i in range(k + 1, n):
            if a[i] > best:
                best, big = a[i], i
        a[k], a[big] = a[big], a[k]
        o[k], o[big] = o[big], o[k]
    return o


def parallel_order(a):
    """dbag_blocks.cu pivot_order_par: ranks (descending, ties by index) and the
    acceptance rule; None = fall back to the selection loop."""
    n = len(a)
    if any(x != x for x in a):
        return None
    o = sorted(range(n), key=lambda i: (-a[i], i))
    for p in range(n - 1):
        x, y, i, j = a[o[p]], a[o[p + 1]], o[p], o[p + 1]
        if not (x > y or (x == y and j == i + 1 and p <= i)):
            return None
    return o


def test_generalized_parallel_pivot_rule():
    """Blocks of D variables with the camera t_x/t_y ties (consecutive indices)."""
    rng = np.random.default_rng(1)
    accepted = 0
    for t in range(4000):
        npt, ncam = int(rng.integers(1, 12)), int(rng.integers(1, 4))
        D = 3 * npt + 6 * ncam
        a = list(rng.uniform(0.5, 2.0, D) * 10.0 ** rng.uniform(-1, 4, D))
        cams = 10.0 ** rng.uniform(0, 6)
        for c in range(ncam):   # cameras: often the largest values, t_x == t_y
            base = 3 * npt + 6 * c
            for m in range(6):
                a[base + m] = cams * rng.uniform(0.1, 10.0)
            a[base + 4] = a[base + 3]
        if t % 5 == 0:          # an accidental tie elsewhere: must fall back or agree
            i, j = rng.integers(0, D, 2)
            a[i] = a[j]
        f = parallel_order(a)
        if f is not None:
            accepted += 1
            assert f == selection_order_n(a), (a, f)
    assert accepted > 1000
