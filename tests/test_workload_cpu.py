"""CPU tests: the synthetic-workload generator against gen_zipf's known answers.

SPEC.md:548-555 (reference /root/reference/SPEC.md) states gen_zipf's contract:
  P(rank k) = k^-s / H_n (inverse CDF over a cumulative table), rank -> key a seeded
  permutation, fully reproducible from the seed; examples: s=0 -> uniform; n=2, s=1 ->
  {2/3, 1/3}; empirical frequencies over 10^6 draws within 3 standard errors per rank
  for the top 100 ranks. paper_2210_08803_b200/workload.py implements it (Zipf, affine_perm).
"""
import numpy as np
import pytest

from paper_2210_08803_b200 import workload as W


def draws(seed, n):
    return W.rng(seed, np.arange(n, dtype=np.uint64))


def test_zipf_s0_is_uniform():
    z = W.Zipf(1000, 0.0)
    assert all(abs(z.prob(k) - 1e-3) < 1e-15 for k in (1, 2, 500, 1000))
    r = z.ranks(draws(0x5EED, 1_000_000))
    f = np.bincount(r, minlength=1000) / 1e6
    se = np.sqrt(1e-3 * (1 - 1e-3) / 1e6)
    assert np.all(np.abs(f - 1e-3) <= 5 * se)  # 1000 ranks: 5 SE keeps the family-wise bound tight


def test_zipf_n2_s1_two_thirds():
    z = W.Zipf(2, 1.0)
    assert z.prob(1) == pytest.approx(2 / 3, abs=1e-15)
    assert z.prob(2) == pytest.approx(1 / 3, abs=1e-15)
    r = z.ranks(draws(0x1234, 1_000_000))
    p1 = np.mean(r == 0)
    assert abs(p1 - 2 / 3) <= 3 * np.sqrt(2 / 9 / 1e6)


@pytest.mark.parametrize("n,s", [(100_000, 1.05), (100_000, 1.1), (10_000, 1.2)])
def test_zipf_top100_within_three_standard_errors(n, s):
    z = W.Zipf(n, s)
    r = z.ranks(draws(0xC0FFEE + n, 1_000_000))
    cnt = np.bincount(r, minlength=n)[:100] / 1e6
    p = np.array([z.prob(k) for k in range(1, 101)])
    se = np.sqrt(p * (1 - p) / 1e6)
    assert np.all(np.abs(cnt - p) <= 3 * se), np.max(np.abs(cnt - p) / se)


def test_zipf_deterministic_and_permuted():
    z = W.Zipf(50_000, 1.1)
    a = z.ranks(draws(7, 10_000))
    b = z.ranks(draws(7, 10_000))
    assert np.array_equal(a, b)
    perm = W.affine_perm(0xABCD, 50_000)
    img = perm(np.arange(50_000))
    assert np.array_equal(np.sort(img), np.arange(50_000))  # a bijection on [0, n)
    assert not np.array_equal(img[:100], np.arange(100))     # hot ranks are not adjacent rows


def test_top_mass_matches_survey_appendix_a4():
    # Zipf top-10% mass s=1.2, 10k of 100k -> 0.9426
    z = W.Zipf(100_000, 1.2)
    assert z.cdf[9_999] / z.H == pytest.approx(0.9426, abs=5e-5)


def test_batchgen_reproducible():
    cfg = W.config3(256)
    g1, g2 = W.BatchGen(cfg, cards=[1000] * 26), W.BatchGen(cfg, cards=[1000] * 26)
    b1, b2 = g1.batch(3), g2.batch(3)
    for x, y in zip(b1 if isinstance(b1, tuple) else (b1,), b2 if isinstance(b2, tuple) else (b2,)):
        assert np.array_equal(np.asarray(x), np.asarray(y))
