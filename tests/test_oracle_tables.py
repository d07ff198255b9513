"""Pins for the histogram (a2) and rule-N1 normalization (a3).

Histogram: brute-force count.  Normalization: the
three SPEC worked examples, the table invariants and
the two tables SURVEY.md 8(c) printed from its own throwaway prototype (g1,
g4), produced with a generator that is restated in synth.lcg_symbols."""
import numpy as np
import pytest

import synth


def test_histogram_bruteforce(orc):
    rng = np.random.default_rng(0)
    s = rng.integers(0, 256, size=100_003).astype(np.uint8)
    assert np.array_equal(orc.histogram(s), np.bincount(s, minlength=256))
    # sample limit: only the leading symbols count
    assert np.array_equal(orc.histogram(s, 1000), np.bincount(s[:1000], minlength=256))
    assert orc.histogram(np.zeros(0, np.uint8)).sum() == 0
    ex = orc.histogram(np.array([0x7F, 0x7F, 0x7F, 0x80], np.uint8))
    assert ex[0x7F] == 3 and ex[0x80] == 1 and ex.sum() == 4


def test_normalize_spec_examples(orc):
    cnt = np.zeros(256, np.uint32)
    cnt[0x7F] = 12345
    f = orc.normalize(cnt)
    assert f[0x7F] == 4096 - 255 and np.all(np.delete(f, 0x7F) == 1)
    cnt = np.zeros(256, np.uint32)
    cnt[3] = cnt[200] = 777
    f = orc.normalize(cnt)
    assert f[3] == 1921 and f[200] == 1921 and f.sum() == 4096
    assert np.all(orc.normalize(np.zeros(256, np.uint32)) == 16)


def test_normalize_invariants_random(orc):
    rng = np.random.default_rng(1)
    for trial in range(400):
        k = rng.integers(1, 257)
        cnt = np.zeros(256, np.uint64)
        idx = rng.choice(256, size=k, replace=False)
        cnt[idx] = rng.integers(0, 10 ** rng.integers(1, 9), size=k)
        if cnt.sum() == 0:
            continue
        f = orc.normalize(cnt.astype(np.uint32)).astype(np.int64)
        assert f.sum() == 4096 and f.min() >= 1
        # proportionality: within one unit of the scaled count, except the
        # symbol that absorbs the remainder (< 256 extra)
        T = cnt.sum()
        ideal = 1 + cnt.astype(np.float64) * 3840 / T
        dev = f - ideal
        best = int(np.argmax(cnt))
        assert np.all(np.delete(dev, best) <= 0) and np.all(np.delete(dev, best) > -1)
        assert -1 < dev[best] < 256
        # monotone in the counts
        order = np.lexsort((-np.arange(256), cnt))  # ties: the lowest symbol last
        assert np.all(np.diff(f[order]) >= 0)


def test_survey_micro_vector_tables(orc):
    """SURVEY.md 8(c) g1 (B=4096, seed 12345) and g4 (B=64, seed 7) tables."""
    g1 = {0x70: 1, 0x72: 2, 0x74: 4, 0x75: 5, 0x76: 5, 0x77: 23, 0x78: 32, 0x79: 59, 0x7A: 118,
          0x7B: 234, 0x7C: 491, 0x7D: 936, 0x7E: 1943}
    f = orc.normalize(orc.histogram(synth.lcg_symbols(4096, 12345)))
    for s in range(256):
        assert f[s] == g1.get(s, 1), hex(s)
    g4 = {0x76: 61, 0x7A: 121, 0x7B: 361, 0x7C: 421, 0x7D: 1081, 0x7E: 1801}
    f = orc.normalize(orc.histogram(synth.lcg_symbols(64, 7)))
    for s in range(256):
        assert f[s] == g4.get(s, 1), hex(s)
