"""Pins of the seeded input generator (gen/): determinism, slice independence,
agreement of its log/cos with libm, and the distributions BASELINE.json asks
for (U,V ~ N(0,1)/sqrt(m_l), D ~ N(0,1)/8, x ~ U[-1,1]); DESIGN.md §3."""
import math

import numpy as np
import pytest

from gen import hgen
from gen.hgen import CONFIGS, HConfig, TAG_D, TAG_U, TAG_V


def test_log_matches_libm():
    rng = np.random.default_rng(1)
    us = np.concatenate([rng.random(2000), [2.0 ** -53, 1e-300, 0.5, 0.7071067811865476, 1.0 - 2 ** -53]])
    for u in us:
        if u <= 0:
            continue
        ref = math.log(u)
        assert abs(hgen.hgen_log(float(u)) - ref) <= 4e-16 * max(1.0, abs(ref))


def test_cos2pi_matches_libm():
    rng = np.random.default_rng(2)
    us = np.concatenate([rng.random(2000), [0.0, 0.25, 0.5, 0.75, 1.0, 1e-9]])
    for u in us:
        assert abs(hgen.hgen_cos2pi(float(u)) - math.cos(2 * math.pi * u)) <= 2e-15


def test_deterministic_and_slice_independent():
    cfg = HConfig("t", d=2, L=2, b=8, r=3, seed=77)
    a = hgen.panel(cfg, TAG_U, 2)
    b = hgen.panel(cfg, TAG_U, 2)
    assert np.array_equal(a, b)
    s = hgen.panel(cfg, TAG_U, 2, 37, 101)
    assert np.array_equal(a[37:101], s)
    x = hgen.xblock(cfg, nrhs=3)
    xs = hgen.xblock(cfg, nrhs=3, row_begin=5, row_end=60)
    assert np.array_equal(x[5:60], xs)
    # a different seed, level, tag or vector gives different numbers
    assert not np.array_equal(a, hgen.panel(cfg, TAG_U, 1))
    assert not np.array_equal(a, hgen.panel(cfg, TAG_V, 2))
    assert not np.array_equal(x, hgen.xblock(cfg, nrhs=3, vec=1))


def test_value_is_panel_entry():
    cfg = CONFIGS["c1"]
    U2 = hgen.panel(cfg, TAG_U, 2, 100, 101)
    for col in (0, 5, cfg.W - 1):
        v = hgen.value(cfg.seed, TAG_U, 2, 0, 100 * cfg.W + col, cfg.lowrank_scale(2))
        assert v == U2[0, col]


def test_distributions():
    cfg = HConfig("t", d=2, L=3, b=64, r=8, seed=5)  # N = 4096, W = 24
    n = cfg.N * cfg.W
    for level in (1, 3):
        p = hgen.panel(cfg, TAG_V, level) * math.sqrt(cfg.m(level))  # back to N(0,1)
        mean, var = p.mean(), p.var()
        assert abs(mean) < 5 / math.sqrt(n)
        assert abs(var - 1.0) < 5 * math.sqrt(2.0 / n)
        # kurtosis of a normal is 3
        k = ((p - mean) ** 4).mean() / var ** 2
        assert abs(k - 3.0) < 0.05
    D = hgen.panel(cfg, TAG_D, 0) * 8.0
    assert abs(D.var() - 1.0) < 5 * math.sqrt(2.0 / D.size)
    x = hgen.xblock(cfg, nrhs=4)
    assert x.min() > -1 and x.max() < 1
    assert abs(x.mean()) < 5 * math.sqrt(1 / 3 / x.size)
    assert abs(x.var() - 1 / 3) < 0.01


def test_config_table_matches_baseline():
    # BASELINE.json configs: N and the "~125 GB" of configs[3]
    assert CONFIGS["c1"].N == 4096 and CONFIGS["c2"].N == 2 ** 20
    assert CONFIGS["c3"].N == 2 ** 21 and CONFIGS["c4"].N == 2 ** 24
    assert CONFIGS["c5"].nrhs == 64
    assert CONFIGS["c4"].factor_bytes == 124_554_051_584
    assert abs(CONFIGS["c4"].factor_bytes / 1e9 - 125) < 1.0
