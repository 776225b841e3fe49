"""Pins of the standard-admissibility oracle (R17):
the paper's interaction counts and load-balance factor, exact tiling, closed
forms and brute force on tiny inputs."""
import numpy as np
import pytest

from gen import hgen
from gen.hgen import HConfig
from oracle import oracle


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def std_panels(d, L, b, r, seed):
    rng = np.random.default_rng(seed)
    c = 1 << d
    N = b * c ** L
    M = 6 ** d - 3 ** d
    U = [rng.standard_normal((N, M * r)) for _ in range(L)]
    V = [rng.standard_normal((N, M * r)) for _ in range(L)]
    Dn = rng.standard_normal((N, 3 ** d * b))
    return U, V, Dn


def morton(d, coords, level):
    k = 0
    for j in range(level):
        for i in range(d):
            k |= ((coords[i] >> j) & 1) << (j * d + i)
    return k


@pytest.mark.parametrize("d", [1, 2, 3])
def test_interaction_counts_and_load_balance(d):
    """an interior level-l box has 3^d 2^d - 3^d admissible
    boxes, a corner box 2^d 2^d - 2^d; the ratio is the load-balance factor
    (3/2)^d."""
    L = {1: 6, 2: 4, 3: 4}[d]
    level = L - 1
    n = 1 << level
    centre = morton(d, [n // 2 - 1] * d, level)   # parent is interior (level >= 3 in 1D/2D)
    corner = morton(d, [0] * d, level)
    _, _, nc = oracle.std_census(d, L, level, centre)
    _, _, nk = oracle.std_census(d, L, level, corner)
    assert nc == 3 ** d * 2 ** d - 3 ** d
    assert nk == 2 ** d * 2 ** d - 2 ** d
    assert nc / nk == pytest.approx((3 / 2) ** d)  # the paper's bound (3/2)^d, attained
    assert oracle.std_slots(d) == 6 ** d - 3 ** d
    # no admissible pair at level 1 (all 2^d children of the root touch)
    assert all(oracle.std_census(d, L, 1, t)[2] == 0 for t in range(1 << d))


@pytest.mark.parametrize("d,L,b", [(1, 4, 2), (2, 3, 1), (2, 3, 2), (3, 2, 1)])
def test_std_tiles_exactly_once(d, L, b):
    cnt = oracle.std_cover_count(d, L, b)
    assert cnt.min() == 1 and cnt.max() == 1


def test_dense_count_is_neighbour_count():
    """Dense blocks = pairs of touching leaves (incl. the diagonal): in 2D with
    n x n leaves, n^2 + 2 n (n-1) * 2 + 2 (n-1)^2 * 2."""
    d, L = 2, 3
    n = 1 << L
    _, dense, _ = oracle.std_census(d, L)
    assert dense == n * n + 4 * n * (n - 1) + 4 * (n - 1) ** 2


@pytest.mark.parametrize("d,L,b,r", [(1, 4, 2, 2), (2, 3, 1, 2), (2, 3, 2, 1), (3, 2, 1, 2), (2, 2, 3, 1)])
def test_std_block_loop_equals_brute_force(d, L, b, r):
    U, V, Dn = std_panels(d, L, b, r, 10 * d + L)
    A = oracle.std_assemble(d, L, b, r, U, V, Dn)
    x = np.random.default_rng(3).standard_normal((len(Dn), 2))
    assert rel(oracle.std_matvec(d, L, b, r, U, V, Dn, x), A @ x) < 1e-13


@pytest.mark.parametrize("d,L,b,r", [(1, 5, 2, 3), (2, 3, 2, 2), (3, 2, 2, 1)])
def test_std_all_ones_closed_form(d, L, b, r):
    """All U, V = 1: every far-field entry equals r, so
    y_i = sum_{j near leaf(i)} D_ij x_j + r sum_{j not near leaf(i)} x_j.
    Catches a missing / extra interaction or a wrong near field."""
    c = 1 << d
    N = b * c ** L
    M = 6 ** d - 3 ** d
    U = [np.ones((N, M * r)) for _ in range(L)]
    V = [np.ones((N, M * r)) for _ in range(L)]
    Dn = np.zeros((N, 3 ** d * b))
    x = np.random.default_rng(4).integers(-8, 9, N).astype(np.float64)
    n = 1 << L
    # leaf coordinates by brute force
    coords = {}
    for k in range(c ** L):
        xc = [0] * d
        for j in range(L):
            for i in range(d):
                xc[i] |= ((k >> (j * d + i)) & 1) << j
        coords[k] = xc
    y = oracle.std_matvec(d, L, b, r, U, V, Dn, x)
    for i in range(0, N, max(1, N // 50)):
        t = i // b
        near = [s for s in range(c ** L) if all(abs(coords[s][q] - coords[t][q]) <= 1 for q in range(d))]
        near_sum = sum(x[s * b:(s + 1) * b].sum() for s in near)
        assert y[i] == pytest.approx(r * (x.sum() - near_sum), abs=1e-12)


def test_std_delta_factor_single_entry():
    """One admissible block (t, s) at level 3 in 2D with U_ts = e_a e_k^T,
    V_ts = e_bb e_k^T gives H = e_{t m + a} e_{s m + bb}^T.  Panel columns use
    slot(t -> s) for U and slot(s -> t) for V (the canonical layout)."""
    d, L, b, r = 2, 3, 2, 2
    N = b * 4 ** L
    M = 27
    level, m = 3, 2
    t = morton(d, [2, 3], level)
    s = morton(d, [5, 4], level)      # parents (1,1) and (2,2): neighbours; boxes 3 apart: admissible
    qt, qs = oracle.std_slot(d, level, t, s), oracle.std_slot(d, level, s, t)
    assert qt >= 0 and qs >= 0
    U = [np.zeros((N, M * r)) for _ in range(L)]
    V = [np.zeros((N, M * r)) for _ in range(L)]
    U[level - 1][t * m + 1, qt * r + 1] = 1.0
    V[level - 1][s * m + 0, qs * r + 1] = 1.0
    A = oracle.std_assemble(d, L, b, r, U, V, np.zeros((N, 9 * b)))
    expect = np.zeros((N, N))
    expect[t * m + 1, s * m + 0] = 1.0
    assert np.array_equal(A, expect)


def test_std_slot_enumeration_is_a_bijection():
    """For every box, slots 0..M-1 are each used exactly once by the in-domain
    and out-of-domain candidates together; in-domain ones are symmetric."""
    d, level = 2, 3
    n = 1 << level
    for t in range(n * n):
        used = []
        for s in range(n * n):
            q = oracle.std_slot(d, level, t, s)
            if q >= 0:
                used.append(q)
                assert oracle.std_slot(d, level, s, t) >= 0
        assert len(set(used)) == len(used) and max(used) < 27


@pytest.mark.parametrize("d,L,b,r", [(1, 4, 2, 2), (2, 3, 1, 2), (2, 3, 2, 1), (3, 2, 1, 2), (2, 2, 3, 1)])
def test_std_transposed_loop_equals_brute_force(d, L, b, r):
    """H^T x by the transposed block loop = A^T x of the assembled matrix (the
    GEMV "T" of PAPER.md:961-969 written out); near-field blocks are not
    symmetric (D_ts != D_st^T), so a loop that forgot to transpose them fails."""
    U, V, Dn = std_panels(d, L, b, r, 20 * d + L)
    A = oracle.std_assemble(d, L, b, r, U, V, Dn)
    x = np.random.default_rng(5).standard_normal((len(Dn), 2))
    assert rel(oracle.std_matvec_t(d, L, b, r, U, V, Dn, x), A.T @ x) < 1e-13
    assert rel(A.T, A) > 1e-3  # the fixture is not symmetric


def test_std_adjoint_identity():
    """<y', H x> = <H^T y', x> between the forward and the transposed loops."""
    d, L, b, r = 2, 4, 4, 3
    U, V, Dn = std_panels(d, L, b, r, 91)
    rng = np.random.default_rng(6)
    x = rng.standard_normal(len(Dn))
    yp = rng.standard_normal(len(Dn))
    lhs = yp @ oracle.std_matvec(d, L, b, r, U, V, Dn, x)
    rhs = oracle.std_matvec_t(d, L, b, r, U, V, Dn, yp) @ x
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def _std_unit_column(d, L, b, r, U, V, Dn, j):
    """H e_j from the definitions (eq:standard-ad-cond on boxes, Def 2.4's
    recursion): at every level l >= 2 the node s = anc_l(j) is the source of a
    low-rank block (t, s) for every box t of the same level that does not touch
    s but whose parent touches s's parent; the near field is the leaves touching
    leaf(j).  Geometry by explicit coordinates; panel columns by the canonical
    slot order (pinned by test_std_slot_enumeration_is_a_bijection)."""
    c = 1 << d
    N = b * c ** L
    M = 6 ** d - 3 ** d
    col = np.zeros(N)
    def coords(k, level):
        x = [0] * d
        for jj in range(level):
            for i in range(d):
                x[i] |= ((k >> (jj * d + i)) & 1) << jj
        return x
    def touch(a, bb):
        return all(abs(a[i] - bb[i]) <= 1 for i in range(d))
    leaf = j // b
    xl = coords(leaf, L)
    for t in range(c ** L):                                  # near field
        xt = coords(t, L)
        if touch(xt, xl):
            e = sum((xl[i] - xt[i] + 1) * 3 ** i for i in range(d))
            col[t * b:(t + 1) * b] += Dn[t * b:(t + 1) * b, e * b + (j - leaf * b)]
    for l in range(2, L + 1):
        m = N // c ** l
        s = j // m
        xs, xps = coords(s, l), coords(s >> d, l - 1)
        for t in range(c ** l):
            xt, xpt = coords(t, l), coords(t >> d, l - 1)
            if touch(xt, xs) or not touch(xpt, xps):
                continue
            qt, qs = oracle.std_slot(d, l, t, s), oracle.std_slot(d, l, s, t)
            v = V[l - 1][j, qs * r:(qs + 1) * r]
            col[t * m:(t + 1) * m] += U[l - 1][t * m:(t + 1) * m, qt * r:(qt + 1) * r] @ v
    assert M * r == U[0].shape[1] if U else True
    return col


@pytest.mark.parametrize("d,L,b,r", [(2, 5, 2, 2), (1, 9, 2, 2), (3, 3, 2, 1)])
def test_std_unit_columns_at_scale(d, L, b, r):
    """Columns of the standard-admissibility H from the definitions vs the
    oracle's block loop, beyond brute-force sizes (N = 1024..2048)."""
    U, V, Dn = std_panels(d, L, b, r, 600 + d + L)
    N = len(Dn)
    js = np.random.default_rng(19).integers(0, N, 6)
    X = np.zeros((N, len(js)))
    X[js, np.arange(len(js))] = 1.0
    Y = oracle.std_matvec(d, L, b, r, U, V, Dn, X)
    for k, j in enumerate(js):
        assert rel(Y[:, k], _std_unit_column(d, L, b, r, U, V, Dn, int(j))) < 1e-13


@pytest.mark.parametrize("cfg", [HConfig("sr2", d=2, L=3, b=4, r=3, adm=1, seed=41),
                                 HConfig("sr3", d=3, L=2, b=2, r=2, adm=1, seed=42),
                                 HConfig("sr1", d=1, L=5, b=3, r=2, adm=1, seed=43),
                                 HConfig("sr0", d=2, L=1, b=5, r=1, adm=1, seed=44)], ids=lambda c: c.name)
def test_std_rows_generated_equals_assembled_matrix(cfg):
    """oracle_std_rows_generated (entries generated on demand, blocks found row
    by row) equals rows of the assembled matrix (brute force) and of the block
    loop, over the seeded panels, at every sampled row."""
    U, V, Dn = hgen.inputs(cfg)
    x = hgen.xblock(cfg, nrhs=2)
    A = oracle.std_assemble(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn)
    rows = np.array(sorted(set([0, cfg.b - 1, cfg.b, cfg.N // 2, cfg.N - 1] + list(range(0, cfg.N, 7)))))
    yr = oracle.std_rows_generated(cfg, x, rows)
    assert rel(yr, (A @ x)[rows]) < 1e-13
    assert rel(yr, oracle.std_matvec(cfg.d, cfg.L, cfg.b, cfg.r, U, V, Dn, x)[rows]) < 1e-13


@pytest.mark.parametrize("d,level", [(1, 3), (1, 6), (2, 3), (2, 4), (3, 3)])
def test_std_slot_order_rederived_from_the_header(d, level):
    """oracle_std_slot against the slot order as include/hmat.h states it,
    re-derived here in plain Python with no call into the oracle: for target t
    (coordinates X, parent P = X >> 1), the candidates are the boxes
    S = 2 (P + eps) + sigma for eps in {-1,0,1}^d, sigma in {0,1}^d, taken in
    increasing (sum_i (eps_i + 1) 3^i) 2^d + sum_i sigma_i 2^i; the ones that
    touch t (every |S_i - X_i| <= 1) are skipped; the others are numbered
    0, 1, ... whether or not they lie inside the domain.  Every ordered pair
    (t, s) of boxes of the level is checked: s gets its number in t's list if it
    is a candidate that does not touch t, else -1 (not in the interaction list:
    eq:standard-ad-cond with the parent-neighbour rule, PAPER.md:279-297,
    615-620).  A dropped out-of-domain candidate, a wrong key order or a wrong
    touch test shifts the numbers and fails here."""
    n = 1 << level

    def coords(k):
        return tuple(sum(((k >> (j * d + i)) & 1) << j for j in range(level)) for i in range(d))

    def morton(xs):
        return sum(((xs[i] >> j) & 1) << (j * d + i) for j in range(level) for i in range(d))

    def eps_list():
        out = [()]
        for _ in range(d):
            out = [e + (v,) for e in out for v in (-1, 0, 1)]
        return out

    M = 6 ** d - 3 ** d
    for t in range(n ** d):
        X = coords(t)
        P = tuple(v >> 1 for v in X)
        keyed = []
        for eps in eps_list():
            for sig in range(1 << d):
                S = tuple(2 * (P[i] + eps[i]) + ((sig >> i) & 1) for i in range(d))
                key = sum((eps[i] + 1) * 3 ** i for i in range(d)) * (1 << d) + sig
                keyed.append((key, S))
        keyed.sort()
        expect = {}
        q = 0
        for _, S in keyed:
            if all(abs(S[i] - X[i]) <= 1 for i in range(d)):
                continue
            if all(0 <= S[i] < n for i in range(d)):
                expect[morton(S)] = q
            q += 1
        assert q == M
        for s in range(n ** d):
            assert oracle.std_slot(d, level, t, s) == expect.get(s, -1), (t, s)


# ---- Def 2.4 read literally (leaf check first) under standard admissibility ----

def _std_counts_closed_form(d, L, strict):
    """Ordered box pairs per level, from the geometry alone: with n = 2^l boxes
    per side, pairs whose parents touch number ((3 n/2 - 2) 4)^d and touching
    pairs (3 n - 2)^d (per dimension 3k - 2 ordered pairs of positions within
    one step among k, then 2 x 2 children per parent pair; dimensions multiply).
    Low rank at level l = parents touch but the boxes do not (eq:standard-ad-cond
    with rho = sqrt(d) on an ideal domain).  Dense blocks: the touching leaf
    pairs (R17), or -- leaf checked first -- every leaf pair whose parents touch."""
    def par(l):
        return ((3 * 2 ** (l - 1) - 2) * 4) ** d

    def touch(l):
        return (3 * 2 ** l - 2) ** d
    if L == 0:
        return 0, 1
    last = L - 1 if strict else L
    lowrank = sum(par(l) - touch(l) for l in range(2, last + 1))
    dense = par(L) if strict else touch(L)
    return lowrank, dense


@pytest.mark.parametrize("d,L", [(1, 1), (1, 4), (1, 7), (2, 1), (2, 2), (2, 3), (2, 5), (3, 2), (3, 3)])
def test_std_census_closed_forms(d, L):
    """Block counts by walking Def 2.4 (both orders) vs the closed forms."""
    assert oracle.std_census(d, L)[:2] == _std_counts_closed_form(d, L, strict=False)
    assert oracle.std_census_strict(d, L) == _std_counts_closed_form(d, L, strict=True)


@pytest.mark.parametrize("d,L,b", [(1, 4, 2), (2, 3, 1), (2, 2, 3), (3, 2, 1)])
def test_std_strict_tiles_exactly_once(d, L, b):
    assert np.all(oracle.std_cover_count_strict(d, L, b) == 1)


@pytest.mark.parametrize("d,L,b,r", [(1, 5, 2, 2), (2, 3, 2, 1), (2, 4, 1, 2), (3, 2, 1, 1), (2, 1, 3, 2)])
def test_std_strict_block_loop_equals_brute_force_and_coarse_structure(d, L, b, r):
    """The literal-order block loop = A x of its assembled matrix; and the
    literal-order structure of depth L, leaf b IS the R17 structure of depth
    L - 1, leaf 2^d b on the same panels (the leaf-level blocks of two touching
    parents tile the parents' near-field block): the two recursions assemble
    the same matrix entry for entry."""
    c = 1 << d
    U, V, _ = std_panels(d, L - 1, c * b, r, 40 + 3 * d + L)
    N = b * c ** L
    Dc = np.random.default_rng(41 + L).standard_normal((N, 3 ** d * c * b))
    A = oracle.std_assemble_strict(d, L, b, r, U, V, Dc)
    assert np.array_equal(A, oracle.std_assemble(d, L - 1, c * b, r, U, V, Dc))
    x = np.random.default_rng(42).standard_normal((N, 2))
    assert rel(oracle.std_matvec_strict(d, L, b, r, U, V, Dc, x), A @ x) < 1e-13
    # the leaf level holds interaction-list pairs as dense blocks: more dense
    # entries than the R17 structure of the same depth and leaf
    lr_s, dn_s = oracle.std_census_strict(d, L)
    lr, dn = oracle.std_census(d, L)[:2]
    assert dn_s >= dn and lr_s <= lr and (L < 2 or dn_s > dn)
