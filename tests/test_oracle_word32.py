"""Pins of the oracle's W = 32 status words (MIS2_FLAG_WORD32; "the same
width as the vertex ids", Eq. 1; reading Q32): Luby on G^2 with the
independently written 32-bit words (Lemma 2), the Fig. 1 replay
with OUT = 2^32 - 1, validity, and the order relation between the 32- and
64-bit priorities that fixes which half of h the short word takes."""
import json
import os
import random

import numpy as np
import pytest

import mis2gen as G
import oracle as O
import pins

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _graphs(count, seed, nmax=50):
    rng = random.Random(seed)
    return [G.random_graph(rng.randrange(1, nmax), rng.choice([0.03, 0.08, 0.2]), seed * 7919 + k,
                           diagonal=rng.random() < 0.5) for k in range(count)]


@pytest.mark.parametrize("chunk", range(2))
def test_luby_on_g2_word32(chunk):
    for g in _graphs(30, 300 + chunk):
        for seed in (0, 99):
            r = O.mis2(g.rowptr, g.colinds, seed=seed, word_bits=32)
            s, it = pins.luby_g2(g.rowptr, g.colinds, seed=seed, word_bits=32)
            assert np.array_equal(r.in_set, s)
            assert r.iterations == it


def test_word32_valid_on_structured_graphs():
    for g in (G.laplace3d_27pt(12), G.elasticity3d(5), G.random_powerlaw_graph(3000, 6, 4)):
        r = O.mis2(g.rowptr, g.colinds, word_bits=32)
        assert pins.is_d2_independent(g.rowptr, g.colinds, r.in_set)
        assert pins.is_d2_maximal(g.rowptr, g.colinds, r.in_set)


def test_word32_words():
    n = 70000  # b = 17: 15 priority bits
    b = O.bits(n)
    rng = np.random.default_rng(3)
    vs = rng.integers(0, n, 400)
    for it in (0, 5):
        w32 = [O.word(it, int(v), n, word_bits=32) for v in vs]
        w64 = [O.word(it, int(v), n) for v in vs]
        assert all(w < (1 << 32) - 1 and (w & ((1 << b) - 1)) == v + 1 for w, v in zip(w32, vs))
        # a smaller 32-bit priority is a smaller 64-bit priority (both are the top bits of h)
        for i in range(len(vs)):
            for j in range(len(vs)):
                if (w32[i] >> b) < (w32[j] >> b):
                    assert (w64[i] >> b) < (w64[j] >> b)


def test_fig1_replay_word32():
    with open(os.path.join(GOLDEN, "fig1.json")) as fh:
        gold = json.load(fh)
    g = G.fig1_graph()
    prio = np.array(gold["priorities"], dtype=np.uint64)
    r = O.mis2(g.rowptr, g.colinds, prio_override=prio, state=True, word_bits=32)
    assert r.M.tolist() == [(1 << 32) - 1] * 6  # OUT of width 32
    assert sorted((np.nonzero(r.in_set)[0] + 1).tolist()) == gold["result_1based"]
    assert r.iterations == gold["iterations"]


def test_aggregation_word32_invariants():
    g = G.laplace3d_7pt(9)
    a = O.aggregate(g.rowptr, g.colinds, word_bits=32)
    r = O.mis2(g.rowptr, g.colinds, word_bits=32)
    assert (a.labels >= 0).all() and a.labels.max() + 1 == a.num_aggs
    # phase-1 roots are the W = 32 MIS-2: each root labels its own aggregate
    roots = np.nonzero(r.in_set)[0]
    assert len(set(a.labels[roots].tolist())) == len(roots)
