"""CPU model of k_column_ring's window search (vx_edt.cu), pinned against the
reference rule it replaces on dense tiles.

edt.py:300-317 returns, for query row q, the FIRST row y minimising
(q - y)^2 + w_y among the candidates.  The kernel evaluates keys
K_y = (w_y << rb) | y, four query rows per block, growing a shared window
by one row on each side per step and stopping once the next distance
squared exceeds every row's current minimum.  This test replays exactly
that arithmetic (u32 keys, clamped edge reads, the incremental squares)
on random columns -- dense, sparse, with rows that have no candidate, and
ragged lengths -- and compares with a brute-force argmin.  CPU only.
"""
import numpy as np
import pytest

M32 = 0xFFFFFFFF


def _keys(w, valid, rb, kinv):
    return [int(kinv) if not v else ((int(x) << rb) | y) for y, (x, v) in enumerate(zip(w, valid))]


def ring_column(w, valid, cap=64, R=4):
    """Winner rows of one column as k_column_ring computes them (None: the
    tile would be handed back to the banded kernel)."""
    L = len(w)
    rb = max(1, (L - 1).bit_length())
    one = 1 << rb
    c = cap + R + 1
    kinv = M32 - ((c * c) << rb)
    K = _keys(w, valid, rb, kinv)
    g = lambda r: K[min(max(r, 0), L - 1)]  # noqa: E731  (clamped shared reads)
    out = []
    for q0 in range(0, L, R):
        k0, k1, k2, k3 = g(q0), g(q0 + 1), g(q0 + 2), g(q0 + 3)
        b = [min(k0, k1 + one, k2 + 4 * one, k3 + 9 * one), min(k0 + one, k1, k2 + one, k3 + 4 * one),
             min(k0 + 4 * one, k1 + one, k2, k3 + one), min(k0 + 9 * one, k1 + 4 * one, k2 + one, k3)]
        o0, o1, o2, o3, d3, steps = one, 4 * one, 9 * one, 16 * one, 9 * one, 0
        more = max(b[0], b[3]) >= o0 or max(b[1], b[2]) >= o1
        while more and steps < cap:   # two steps per trip, as the kernel
            o4 = o3 + d3
            d3 += 2 * one
            s = steps + 1
            kl, kr, kl2, kr2 = g(q0 - s), g(q0 + 3 + s), g(q0 - s - 1), g(q0 + 4 + s)
            offl, offr = (o0, o1, o2, o3), (o3, o2, o1, o0)
            offl2, offr2 = (o1, o2, o3, o4), (o4, o3, o2, o1)
            b = [min(b[i], (kl + offl[i]) & M32, (kr + offr[i]) & M32, (kl2 + offl2[i]) & M32,
                     (kr2 + offr2[i]) & M32) for i in range(4)]
            o0, o1, o2 = o2, o3, o4
            o3 = o4 + d3
            d3 += 2 * one
            steps += 2
            more = max(b[0], b[3]) >= o0 or max(b[1], b[2]) >= o1
        if more:
            return None
        out += [v & (one - 1) for v in b][: max(0, min(R, L - q0))]
    return out


def brute_column(w, valid):
    L = len(w)
    res = []
    for q in range(L):
        best, arg = None, None
        for y in range(L):
            if valid[y]:
                d = (q - y) ** 2 + int(w[y])
                if best is None or d < best:
                    best, arg = d, y
        res.append(arg)
    return res


@pytest.mark.parametrize("L", [1, 2, 3, 5, 24, 33, 64, 97, 512])
@pytest.mark.parametrize("density", [1.0, 0.9, 0.3, 0.05])
def test_ring_model_matches_first_minimiser(L, density):
    rng = np.random.default_rng(L * 7 + int(density * 100))
    for trial in range(6 if L < 512 else 2):
        wmax = int(rng.choice([4, 50, 400, 5000]))
        w = rng.integers(0, wmax + 1, L)
        valid = rng.random(L) < density
        if not valid.any():
            valid[rng.integers(L)] = True
        got = ring_column(w, valid)
        want = brute_column(w, valid)
        if got is None:   # handed back: the banded kernel answers
            continue
        assert got == want, (L, density, trial)


def test_ring_model_ties_pick_lowest_row():
    # equal distances on both sides of every query row: the lowest row wins
    w = np.zeros(40, np.int64)
    valid = np.zeros(40, bool)
    valid[::4] = True
    assert ring_column(w, valid) == brute_column(w, valid)
    w2 = np.array([9, 0, 9, 1, 1, 0, 4, 4, 0, 9] * 5)
    assert ring_column(w2, np.ones(50, bool)) == brute_column(w2, np.ones(50, bool))


def test_ring_model_hands_back_when_no_candidate_in_reach():
    valid = np.zeros(300, bool)
    valid[0] = True
    assert ring_column(np.zeros(300, np.int64), valid, cap=16) is None
