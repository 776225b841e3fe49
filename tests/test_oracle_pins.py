"""Pins of the CPU oracle (oracle/) against things other than itself
(DESIGN.md §5): the paper's worked example, closed forms, special cases that
reduce to textbook routines, invariants, and brute force on tiny inputs.

Each test names the plausible oracle mistake it would catch.
"""
import itertools

import numpy as np
import pytest

from gen import hgen
from gen.hgen import CONFIGS, HConfig
from oracle import oracle

ALL = (1 << 64) - 1


def rand_panels(d, L, b, r, seed):
    """Random canonical panels (numpy generator; the tests' own inputs)."""
    rng = np.random.default_rng(seed)
    c = 1 << d
    N = b * c ** L
    W = (c - 1) * r
    U = [rng.standard_normal((N, W)) for _ in range(L)]
    V = [rng.standard_normal((N, W)) for _ in range(L)]
    D = rng.standard_normal((N, b))
    return U, V, D


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# -- structure ---------------------------------------------------------------

@pytest.mark.parametrize("d,L", [(1, 0), (1, 1), (1, 5), (2, 1), (2, 2), (2, 4), (3, 1), (3, 3)])
def test_block_census_formula(d, L):
    """Counts by walking Def 2.4 vs the closed forms c^{L+1}-c low-rank,
    c^L dense. Catches a wrong recursion/admissibility."""
    c = 1 << d
    lr, dense, lr1 = oracle.block_census(d, L)
    assert lr == c ** (L + 1) - c
    assert dense == c ** L
    assert lr1 == (c * (c - 1) if L >= 1 else 0)


def test_paper_worked_example_12_of_16():
    """in 2D, 12 of the 16 level-1 child pairs are
    admissible (low-rank); the other 4 are H-matrices of their own."""
    lr, dense, lr1 = oracle.block_census(2, 3)
    assert lr1 == 12
    assert 16 - lr1 == 4


@pytest.mark.parametrize("d,L,b", [(1, 3, 2), (2, 2, 4), (2, 3, 1), (3, 1, 8), (3, 2, 1)])
def test_blocks_tile_the_matrix_exactly_once(d, L, b):
    """P8: dense leaf blocks + all sibling blocks cover every (i, j) exactly
    once.  Catches a missing or doubled block."""
    cnt = oracle.cover_count(d, L, b)
    assert cnt.min() == 1 and cnt.max() == 1


def test_storage_formula_matches_baseline():
    """PAPER.md:390-394 O(rN log N); exact N(2(c-1)rL + b) scalars.  BASELINE
    quotes "~125 GB of factors" for configs[3]."""
    assert CONFIGS["c4"].factor_bytes == 8 * (2 ** 24) * (2 * 3 * 16 * 9 + 64)
    assert 124e9 < CONFIGS["c4"].factor_bytes < 125e9
    assert CONFIGS["c1"].factor_bytes == 6_815_744


def test_sibling_slot_maps():
    """Siblings: the other children of the parent, ascending, never self;
    slot() inverts sibling()."""
    for c in (2, 4, 8):
        for t in range(3 * c):
            sibs = [oracle.sibling(c, t, q) for q in range(c - 1)]
            assert sibs == [p for p in range((t // c) * c, (t // c) * c + c) if p != t]
            for q, s in enumerate(sibs):
                assert oracle.slot(c, t, s) == q
                assert oracle.sibling(c, s, oracle.slot(c, s, t)) == t


# -- closed forms and special cases --------------------------------------------

def test_d1_L1_b1_r1_closed_form():
    """H = [[D0, u01 v01], [u10 v10, D1]] (Def 2.4 with one level).  Panel
    rows: U_1[0] = U_{0,1}, U_1[1] = U_{1,0}; V_1[0] = V_{1,0} (source 0),
    V_1[1] = V_{0,1} (source 1).  Catches U/V or t/s transposition."""
    U = [np.array([[2.0], [3.0]])]
    V = [np.array([[5.0], [7.0]])]
    D = np.array([[11.0], [13.0]])
    H = np.array([[11.0, 2.0 * 7.0], [3.0 * 5.0, 13.0]])
    x = np.array([0.5, -1.25])
    assert np.array_equal(oracle.matvec(1, 1, 1, 1, U, V, D, x), H @ x)
    assert np.array_equal(oracle.assemble(1, 1, 1, 1, U, V, D), H)


@pytest.mark.parametrize("d,L,b,r", [(1, 2, 3, 2), (2, 2, 4, 2), (3, 1, 2, 3), (2, 3, 2, 1)])
def test_delta_factor_gives_single_entry(d, L, b, r):
    """A rank-1 delta block: U_{t,s} = e_a e_k^T, V_{t,s} = e_bb e_k^T gives
    H = e_{t m + a} e_{s m + bb}^T.  The panel positions follow
    the canonical layout: U_l row t m + a, column slot(t->s) r + k;
    V_l row s m + bb, column slot(s->t) r + k.  Catches a wrong slot mapping."""
    c = 1 << d
    N = b * c ** L
    W = (c - 1) * r
    rng = np.random.default_rng(d * 100 + L)
    for _ in range(4):
        level = int(rng.integers(1, L + 1))
        m = N // c ** level
        t = int(rng.integers(0, c ** level))
        par = t // c
        s = int(rng.choice([p for p in range(par * c, par * c + c) if p != t]))
        a, bb, k = int(rng.integers(0, m)), int(rng.integers(0, m)), int(rng.integers(0, r))
        q_ts = sorted(p for p in range(par * c, par * c + c) if p != t).index(s)
        q_st = sorted(p for p in range(par * c, par * c + c) if p != s).index(t)
        U = [np.zeros((N, W)) for _ in range(L)]
        V = [np.zeros((N, W)) for _ in range(L)]
        U[level - 1][t * m + a, q_ts * r + k] = 1.0
        V[level - 1][s * m + bb, q_st * r + k] = 1.0
        D = np.zeros((N, b))
        A = oracle.assemble(d, L, b, r, U, V, D)
        expect = np.zeros((N, N))
        expect[t * m + a, s * m + bb] = 1.0
        assert np.array_equal(A, expect)
        x = rng.standard_normal(N)
        y = oracle.matvec(d, L, b, r, U, V, D, x)
        assert np.array_equal(y, expect @ x)


@pytest.mark.parametrize("d,L,b,r", [(1, 4, 2, 3), (2, 3, 4, 2), (3, 2, 2, 1), (2, 2, 64, 8)])
def test_all_ones_factors_closed_form(d, L, b, r):
    """All U, V entries = 1: every sibling block is r * ones, so every entry
    outside the leaf-diagonal blocks of H equals r:
        y_i = (D x)_i + r (sum_j x_j - sum_{j in leaf(i)} x_j).
    Catches a dropped level, a wrong node range m_l or a missing sibling."""
    c = 1 << d
    N = b * c ** L
    W = (c - 1) * r
    U = [np.ones((N, W)) for _ in range(L)]
    V = [np.ones((N, W)) for _ in range(L)]
    rng = np.random.default_rng(3)
    D = rng.standard_normal((N, b))
    x = rng.integers(-8, 9, N).astype(np.float64)  # small integers: exact sums
    leaf_sum = x.reshape(-1, b).sum(axis=1).repeat(b)
    Dx = np.einsum("kij,kj->ki", D.reshape(-1, b, b), x.reshape(-1, b)).reshape(-1)
    y = oracle.matvec(d, L, b, r, U, V, D, x)
    assert rel(y, Dx + r * (x.sum() - leaf_sum)) < 1e-14


@pytest.mark.parametrize("d,b", [(1, 5), (2, 7), (3, 16)])
def test_depth0_is_plain_gemv(d, b):
    """L = 0: the root is a leaf, H = D_0 (a b x b dense GEMV)."""
    rng = np.random.default_rng(4)
    D = rng.standard_normal((b, b))
    x = rng.standard_normal((b, 3))
    y = oracle.matvec(d, 0, b, 2, [], [], D, x)
    assert rel(y, D @ x) < 1e-15


def test_zero_factors_block_diagonal_and_zero_x():
    """U = V = 0 gives the block-diagonal GEMV; x = 0 gives y = 0."""
    d, L, b, r = 2, 2, 4, 3
    U, V, D = rand_panels(d, L, b, r, 5)
    Z = [np.zeros_like(u) for u in U]
    rng = np.random.default_rng(6)
    x = rng.standard_normal(len(D))
    y = oracle.matvec(d, L, b, r, Z, Z, D, x)
    expect = np.einsum("kij,kj->ki", D.reshape(-1, b, b), x.reshape(-1, b)).reshape(-1)
    assert rel(y, expect) < 1e-15
    assert np.array_equal(oracle.matvec(d, L, b, r, U, V, D, np.zeros_like(x)), np.zeros_like(x))


# -- brute force ----------------------------------------------------------------

GRID = [(d, L, b, r) for d, L, b, r in itertools.product((1, 2, 3), (0, 1, 2, 3), (1, 4, 8), (1, 2, 8))
        if b * (1 << d) ** L <= 512]


@pytest.mark.parametrize("d,L,b,r", GRID)
def test_block_loop_equals_brute_force(d, L, b, r):
    """Block loop vs numpy's dense product of the assembled matrix (P3)."""
    U, V, D = rand_panels(d, L, b, r, d * 1000 + L * 100 + b * 10 + r)
    A = oracle.assemble(d, L, b, r, U, V, D)
    rng = np.random.default_rng(7)
    x = rng.standard_normal((len(D), 2))
    y = oracle.matvec(d, L, b, r, U, V, D, x)
    assert rel(y, A @ x) < 1e-13
    assert rel(oracle.dense_matvec(A, x), A @ x) < 1e-14


def test_assembly_matches_textbook_blocks():
    """Assembled block (t, s) equals U_ts @ V_ts^T formed with numpy from the
    panel slices (layout of DESIGN.md §4), for every block of a 2D L=2 case."""
    d, L, b, r = 2, 2, 2, 3
    c, N, W = 4, 2 * 16, 9
    U, V, D = rand_panels(d, L, b, r, 8)
    A = oracle.assemble(d, L, b, r, U, V, D)
    for level in (1, 2):
        m = N // c ** level
        for t in range(c ** level):
            par = t // c
            sibs = [p for p in range(par * c, par * c + c) if p != t]
            for q, s in enumerate(sibs):
                qs = [p for p in range(par * c, par * c + c) if p != s].index(t)
                Uts = U[level - 1][t * m:(t + 1) * m, q * r:(q + 1) * r]
                Vts = V[level - 1][s * m:(s + 1) * m, qs * r:(qs + 1) * r]
                assert np.allclose(A[t * m:(t + 1) * m, s * m:(s + 1) * m], Uts @ Vts.T, rtol=0, atol=1e-14)
    for k in range(N // b):
        assert np.array_equal(A[k * b:(k + 1) * b, k * b:(k + 1) * b], D[k * b:(k + 1) * b])


def test_c1_brute_force_assembled_4096():
    """BASELINE configs[0]: C1 checked against a dense brute-force matvec of the
    assembled 4096 x 4096 matrix, on the seeded synthetic inputs."""
    cfg = CONFIGS["c1"]
    U, V, D = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=1)
    A = oracle.assemble(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D)
    y = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
    assert rel(y, oracle.dense_matvec(A, x)) < 1e-13
    # extended-precision reference of the same assembled matrix
    Ax = (A.astype(np.longdouble) @ x.astype(np.longdouble)).astype(np.float64)
    assert rel(y, Ax) < 1e-14


# -- linearity, superposition -----------------------------------------------------

def test_linearity_superposition_and_columns():
    """H(ax + bx') = aHx + bHx'; y = y_D + sum_l y_l over level masks; the
    columns of a multi-RHS call equal single-vector calls (P4)."""
    d, L, b, r = 2, 3, 4, 2
    U, V, D = rand_panels(d, L, b, r, 9)
    N = len(D)
    rng = np.random.default_rng(10)
    x1, x2 = rng.standard_normal(N), rng.standard_normal(N)
    H = lambda v: oracle.matvec(d, L, b, r, U, V, D, v)
    assert rel(H(2.5 * x1 - 0.75 * x2), 2.5 * H(x1) - 0.75 * H(x2)) < 1e-14
    parts = oracle.matvec(d, L, b, r, U, V, D, x1, level_mask=0, dense=True)
    for level in range(1, L + 1):
        parts = parts + oracle.matvec(d, L, b, r, U, V, D, x1, level_mask=1 << (level - 1), dense=False)
    assert rel(parts, H(x1)) < 1e-14
    X = np.stack([x1, x2], axis=1)
    Y = oracle.matvec(d, L, b, r, U, V, D, X)
    assert np.array_equal(Y[:, 0], H(x1)) and np.array_equal(Y[:, 1], H(x2))


# -- the sampled-rows oracle ---------------------------------------------------------

@pytest.mark.parametrize("cfg", [CONFIGS["c1"], HConfig("t3", d=3, L=2, b=8, r=4, seed=11),
                                 HConfig("t1", d=1, L=6, b=4, r=3, seed=12)])
def test_rows_generated_equals_block_loop(cfg):
    """oracle_rows_generated (factors generated on demand) equals the block
    loop over fully generated panels at every sampled row."""
    U, V, D = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=2)
    y = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
    rows = np.array(sorted(set([0, 1, cfg.b - 1, cfg.b, cfg.N // 2, cfg.N - 1] + list(range(0, cfg.N, 37)))))
    yr = oracle.rows_generated(cfg, x, rows)
    assert rel(yr, y[rows]) < 1e-13


# -- transposed product (GEMV "T") -------------------------------

@pytest.mark.parametrize("d,L,b,r", [(1, 3, 2, 2), (2, 2, 4, 3), (3, 1, 8, 2), (2, 3, 3, 1), (1, 0, 5, 2)])
def test_transpose_block_loop_equals_brute_force(d, L, b, r):
    """oracle.matvec_t = A^T x with A the assembled matrix (brute force)."""
    U, V, D = rand_panels(d, L, b, r, 60 + d + L)
    A = oracle.assemble(d, L, b, r, U, V, D)
    x = np.random.default_rng(61).standard_normal((len(D), 2))
    assert rel(oracle.matvec_t(d, L, b, r, U, V, D, x), A.T @ x) < 1e-13


# -- the paper-strict reading of Def 2.4 (R1) -----------------

@pytest.mark.parametrize("d,L", [(1, 1), (1, 4), (2, 1), (2, 2), (2, 3), (3, 2)])
def test_strict_census(d, L):
    """Leaves checked first: every child pair of a leaf-parent is dense, so
    low-rank blocks live at levels 1..L-1 (c^L - c of them) and c^{L+1} dense
    b x b blocks tile the leaf-parent diagonal."""
    c = 1 << d
    lr, dense, lr1 = oracle.block_census_strict(d, L)
    assert lr == c ** L - c
    assert dense == c ** (L + 1)
    if d == 2 and L >= 2:
        assert lr1 == 12  # the paper's walkthrough: 12 of 16
    if L == 1:
        assert lr1 == 0   # the root's children are leaves: all pairs dense


@pytest.mark.parametrize("d,L,b", [(1, 3, 2), (2, 2, 2), (3, 2, 1), (2, 1, 3)])
def test_strict_tiles_exactly_once(d, L, b):
    cnt = oracle.cover_count_strict(d, L, b)
    assert cnt.min() == 1 and cnt.max() == 1


def test_strict_storage_matches_survey():
    """8 [2(c-1) r N (L-1) + N c b] bytes: 137.44 GB for configs[3]'s shape, vs
    124.55 GB for the BASELINE reading (the survey's byte check of R1)."""
    c, r, N, L, b = 4, 16, 2 ** 24, 9, 64
    assert 8 * (2 * (c - 1) * r * N * (L - 1) + N * c * b) == 137_438_953_472


@pytest.mark.parametrize("d,L,b,r", [(1, 3, 2, 2), (2, 2, 2, 3), (3, 2, 1, 2), (2, 3, 4, 1)])
def test_strict_block_loop_brute_force_and_equivalence(d, L, b, r):
    """Strict block loop = brute force of the strict assembled matrix, and the
    strict H-matrix of depth L, leaf b is the BASELINE-reading H-matrix of
    depth L-1, leaf 2^d b on the same panels (what hmat_create_strict uses)."""
    c = 1 << d
    N = b * c ** L
    W = (c - 1) * r
    rng = np.random.default_rng(70 + d * 10 + L)
    U = [rng.standard_normal((N, W)) for _ in range(L - 1)]
    V = [rng.standard_normal((N, W)) for _ in range(L - 1)]
    Dc = rng.standard_normal((N, c * b))
    x = rng.standard_normal((N, 2))
    A = oracle.assemble_strict(d, L, b, r, U, V, Dc)
    y = oracle.matvec_strict(d, L, b, r, U, V, Dc, x)
    assert rel(y, A @ x) < 1e-13
    assert rel(oracle.matvec(d, L - 1, c * b, r, U, V, Dc, x), y) < 1e-14


def unit_column(d, L, b, r, U, V, D, j):
    """H e_j written straight from the block structure, in
    O(N r) without the oracle's loops: the dense leaf block of j's leaf gives
    column j mod b of D_leaf in that leaf's rows; at every level l the node
    s = anc_l(j) is the SOURCE of the blocks (t, s) for each sibling t of s, whose
    column j is U_ts V_ts[j - s m_l, :]^T in t's rows.  Panel addressing per
    include/hmat.h: U_l row i, slot q = sibling q of t (target-major); V_l row j,
    slot q' = sibling q' of s, i.e. the target (source-major)."""
    c = 1 << d
    N = b * c ** L
    col = np.zeros(N)
    k = j // b
    col[k * b:(k + 1) * b] += D[k * b:(k + 1) * b, j - k * b]
    for l in range(1, L + 1):
        m = N // c ** l
        s = j // m
        me = s % c
        for qp in range(c - 1):                     # targets t = siblings of s, V slot qp
            t = (s // c) * c + (qp if qp < me else qp + 1)
            q = me if me < t % c else me - 1        # slot of s in t's list (U's column block)
            v = V[l - 1][j, qp * r:(qp + 1) * r]
            col[t * m:(t + 1) * m] += U[l - 1][t * m:(t + 1) * m, q * r:(q + 1) * r] @ v
    return col


@pytest.mark.parametrize("d,L,b,r", [(2, 6, 16, 4), (3, 4, 8, 3), (1, 12, 4, 2)])
def test_unit_columns_at_scale(d, L, b, r):
    """Columns of H from the definition vs the oracle's block loop on unit
    vectors, at N = 2^14..2^16 (beyond brute-force assembly): catches a slot map
    or node range that is only wrong away from the tiny shapes."""
    U, V, D = rand_panels(d, L, b, r, 500 + d + L)
    N = len(D)
    rng = np.random.default_rng(17)
    js = rng.integers(0, N, 12)
    X = np.zeros((N, len(js)))
    X[js, np.arange(len(js))] = 1.0
    Y = oracle.matvec(d, L, b, r, U, V, D, X)
    for k, j in enumerate(js):
        assert rel(Y[:, k], unit_column(d, L, b, r, U, V, D, int(j))) < 1e-14


# -- the all-cores block loop and its generated-factor form (full-size parity) --

@pytest.mark.parametrize("d,L,b,r", [(1, 5, 3, 2), (2, 3, 4, 3), (2, 4, 8, 2), (3, 2, 4, 2), (2, 0, 5, 2)])
@pytest.mark.parametrize("nrhs", [1, 3])
def test_matvec_par_bitwise_equals_block_loop(d, L, b, r, nrhs):
    """oracle_matvec_rows_par does the block loop's arithmetic element for
    element in the same order, only split over threads: bit-identical to
    `matvec` for any thread count, any row range and any level selection.  A
    dropped level, a wrong z (t/s or slot transposition), a race or an
    off-by-one in the row range shows as a bit difference."""
    U, V, D = rand_panels(d, L, b, r, 1000 + 7 * d + L)
    N = len(D)
    x = np.random.default_rng(77).standard_normal((N, nrhs))
    ref = oracle.matvec(d, L, b, r, U, V, D, x)
    for th in (1, 3, 8):
        assert np.array_equal(oracle.matvec_par(d, L, b, r, U, V, D, x, threads=th), ref)
    for r0, r1 in [(0, N // 3), (N // 3, N - 1), (min(b + 1, N - 2), min(b + 2, N - 1)), (N - 1, N)]:
        got = oracle.matvec_par(d, L, b, r, U, V, D, x, threads=4, row_begin=r0, row_end=r1)
        assert np.array_equal(got, ref[r0:r1])
    if L >= 2:
        mask = 0b10
        assert np.array_equal(oracle.matvec_par(d, L, b, r, U, V, D, x, level_mask=mask, dense=False),
                              oracle.matvec(d, L, b, r, U, V, D, x, level_mask=mask, dense=False))


@pytest.mark.parametrize("cfg", [CONFIGS["c1"], HConfig("g3", d=3, L=2, b=8, r=3, seed=71),
                                 HConfig("g1", d=1, L=6, b=4, r=5, seed=72),
                                 HConfig("gs", d=2, L=2, b=256, r=16, seed=73)], ids=lambda c: c.name)
@pytest.mark.parametrize("nrhs", [1, 2, 64])
def test_matvec_generated_bitwise_equals_block_loop(cfg, nrhs):
    """The generated-factor form (the full-size parity oracle) equals the block
    loop run on the panels hgen writes, bit for bit, so the pins of the block
    loop carry over to it; any row range gives the same rows."""
    U, V, D = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=nrhs, vec=2)
    ref = oracle.matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, D, x)
    assert np.array_equal(oracle.matvec_generated(cfg, x, threads=5), ref)
    r0, r1 = cfg.N // 4 + 3, cfg.N // 2 + 1
    assert np.array_equal(oracle.matvec_generated(cfg, x, r0, r1, threads=2), ref[r0:r1])
