"""Pins the C restatement (oracle/liboracle.so) against the UNMODIFIED reference.

The reference side runs the real specsim headers compiled in place
(oracle/_ref/libspecsim_ref.so, see oracle/Makefile and oracle/ref_bridge.cpp).
Every comparison is bit-exact: same tokens, same parents, same fp64 path
probabilities, same RNG words, same bandit picks.
"""
import ctypes as C
import itertools
import random

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="reference bridge not built")


def _arr(t, n):
    return (t * n)()


# ------------------------------------------------------------------ RNG
@pytest.mark.parametrize("seed,stream", [(0, 0), (1, 0), (42, 7), (2**63 + 5, 0x52515254 + 3), (399, 77)])
def test_rng_streams_match(seed, stream):
    R, L = O.ref(), O.orc()
    r = R.ref_rng_create(seed, stream)
    o = O.Rng(seed, stream)
    try:
        for i in range(700):  # > 2 mt19937_64 twists
            assert R.ref_rng_next_u64(r) == o.next_u64()
        for i in range(50):
            assert R.ref_rng_uniform01(r) == o.uniform01()
            n = 1 + i * 7
            assert R.ref_rng_uniform_int(r, n) == o.uniform_int(n)
            assert R.ref_rng_normal(r) == o.normal()
        for label in [0, 1, 0x53454C, 0x52515254 + 9, 2**40 + 3]:
            rf = R.ref_rng_fork(r, label)
            of = o.fork(label)
            for _ in range(20):
                assert R.ref_rng_next_u64(rf) == of.next_u64()
            R.ref_rng_destroy(rf)
    finally:
        R.ref_rng_destroy(r)


# ------------------------------------------------------- distributions
def _rows(seed, v, n, ties=True):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        x = rng.integers(0, 5, size=v).astype(np.float64) if ties else rng.random(v)
        x[rng.random(v) < 0.2] = 0.0
        if x.sum() == 0:
            x[0] = 1.0
        out.append(x / x.sum())
    return out


def test_argmax_inverse_cdf_temper_match():
    R, L = O.ref(), O.orc()
    L.orc_argmax.argtypes = [C.c_void_p, C.c_int]
    L.orc_inverse_cdf_pick.argtypes = [C.c_void_p, C.c_int, C.c_double]
    L.orc_temper.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_void_p]
    for row in _rows(3, 37, 40):
        p = row.ctypes.data_as(C.c_void_p)
        assert R.ref_argmax(p, 37) == L.orc_argmax(p, 37)
        for u in [0.0, 1e-12, 0.3, 0.5, 0.999999, float(np.nextafter(1.0, 0))] + list(np.cumsum(row)[:5]):
            assert R.ref_inverse_cdf_pick(p, 37, u) == L.orc_inverse_cdf_pick(p, 37, u)
        for t in [0.0, 1.0, 0.5, 0.9, 2.0]:
            a = np.zeros(37)
            b = np.zeros(37)
            assert R.ref_target_next_dist(p, 37, t, a.ctypes.data_as(C.c_void_p)) == 0
            L.orc_temper(p, 37, t, b.ctypes.data_as(C.c_void_p))
            assert np.array_equal(a, b)


def test_strategy_capacity_sweep():
    R, L = O.ref(), O.orc()
    L.orc_strategy_validate.argtypes = [C.c_void_p, C.c_void_p]
    for d, k, t in itertools.product(range(0, 11), range(0, 9), [1, 3, 8, 16, 32, 64, 128, 340, 1000]):
        s = O.Strategy(d, k, t)
        assert R.ref_max_tree_nodes(d, k, t) == L.orc_max_tree_nodes(C.byref(s))
        assert (R.ref_strategy_validate(d, k, t) == 0) == (L.orc_strategy_validate(C.byref(s), None) == 0)


# ---------------------------------------------------------------- tree
def _tree_ref(user, v, ctx, d, k, t):
    R = O.ref()
    n = t
    tok, par, dep = _arr(C.c_int32, n), _arr(C.c_int32, n), _arr(C.c_int32, n)
    prob, pp = _arr(C.c_double, n), _arr(C.c_double, n)
    cctx = (C.c_int32 * max(1, len(ctx)))(*ctx)
    got = R.ref_build_draft_tree(O.fnptr(O.orc(), "orc_test_row"), C.byref(user), v, cctx, len(ctx), d, k, t,
                                 tok, par, dep, prob, pp)
    assert got >= 0
    return [(tok[i], par[i], dep[i], prob[i], pp[i]) for i in range(got)]


def _tree_orc(user, v, d, k, t):
    L = O.orc()
    L.orc_build_draft_tree.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    out = (O.Node * t)()
    s = O.Strategy(d, k, t)
    got = L.orc_build_draft_tree(O.fnptr(L, "orc_test_row"), C.byref(user), v, C.byref(s), out)
    assert got >= 0
    return [(out[i].token, out[i].parent, out[i].depth, out[i].prob, out[i].path_prob) for i in range(got)]


CASES = [(v, d, k, t, lv, z) for (v, d, k, t) in [(6, 4, 2, 8), (3, 4, 3, 8), (8, 4, 2, 8), (16, 4, 4, 16),
                                                   (32, 6, 8, 16), (50, 10, 8, 64), (7, 3, 1, 3), (40, 5, 3, 30),
                                                   (64, 8, 8, 128), (5, 2, 5, 30)]
         for (lv, z) in [(0, 0), (3, 20), (2, 50), (6, 0)]]


@pytest.mark.parametrize("v,d,k,t,levels,zero_pct", CASES)
def test_build_draft_tree_matches_reference(v, d, k, t, levels, zero_pct):
    if t > O.orc().orc_max_tree_nodes(C.byref(O.Strategy(d, k, t))):
        pytest.skip("invalid strategy")
    for seed in range(4):
        user = O.TestRows(1000 * seed + v + d * 7 + k * 13 + t, v, levels, zero_pct)
        a = _tree_ref(user, v, [2, 5, 1], d, k, t)
        b = _tree_orc(user, v, d, k, t)
        assert a == b


@pytest.mark.parametrize("v,d,k,t,levels,zero_pct", CASES[::3])
def test_verify_greedy_matches_reference(v, d, k, t, levels, zero_pct):
    R, L = O.ref(), O.orc()
    if t > L.orc_max_tree_nodes(C.byref(O.Strategy(d, k, t))):
        pytest.skip("invalid strategy")
    L.orc_verify_greedy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    for seed in range(6):
        drafter = O.TestRows(seed * 31 + 1, v, levels, zero_pct)
        tree = _tree_orc(drafter, v, d, k, t)
        # target rows: a different keyed family; with few levels the drafter's
        # top choices match the target's argmax often enough to walk deep
        target = O.TestRows(seed * 31 + 1 if seed % 2 == 0 else seed * 977 + 5, v, levels, zero_pct)
        n = len(tree)
        tok = (C.c_int32 * n)(*[x[0] for x in tree])
        par = (C.c_int32 * n)(*[x[1] for x in tree])
        acc = _arr(C.c_int32, 64)
        alen, bonus = C.c_int32(), C.c_int32()
        ctx = (C.c_int32 * 2)(3, 4)
        assert R.ref_verify_greedy(O.fnptr(L, "orc_test_row"), C.byref(target), v, ctx, 2, n, tok, par, acc,
                                   C.byref(alen), C.byref(bonus)) == 0
        nodes = (O.Node * n)()
        for i, x in enumerate(tree):
            nodes[i] = O.Node(*x)
        res = O.Accept()
        assert L.orc_verify_greedy(O.fnptr(L, "orc_test_argmax"), C.byref(target), nodes, n, C.byref(res)) == 0
        assert res.accept_length == alen.value
        assert res.bonus == bonus.value
        assert list(res.accepted[:alen.value]) == list(acc[:alen.value])
        for j in range(alen.value):  # accepted node indices walk parent links
            nd = res.nodes[j]
            assert tree[nd][0] == res.accepted[j]
            assert tree[nd][1] == (res.nodes[j - 1] if j else -1)


@pytest.mark.parametrize("temperature", [1.0, 0.9, 0.5])
@pytest.mark.parametrize("v,depth", [(8, 3), (5, 1), (64, 6), (4, 8)])
def test_sampled_chain_and_stochastic_verify_match(temperature, v, depth):
    R, L = O.ref(), O.orc()
    L.orc_build_sampled_chain.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                          C.c_void_p]
    L.orc_verify_stochastic.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_void_p, C.c_int,
                                        C.c_void_p, C.c_void_p, C.c_void_p]
    row = O.fnptr(L, "orc_test_row")
    for seed in range(25):
        drafter = O.TestRows(seed + 11, v, 4 if seed % 2 else 0, 10 * (seed % 3))
        target = O.TestRows(seed + 11 if seed % 4 == 0 else seed + 500, v, 4 if seed % 3 else 0, 10 * (seed % 2))
        rr = R.ref_rng_create(seed, 0x52515254 + seed)
        ro = O.Rng(seed, 0x52515254 + seed)
        ctx = (C.c_int32 * 1)(2)
        tok, prob, pp = _arr(C.c_int32, depth), _arr(C.c_double, depth), _arr(C.c_double, depth)
        dd_ref = np.zeros(depth * v)
        assert R.ref_build_sampled_chain(row, C.byref(drafter), v, ctx, 1, depth, rr, tok, prob, pp,
                                         dd_ref.ctypes.data_as(C.c_void_p)) == depth
        chain = (O.Node * depth)()
        dd = np.zeros(depth * v)
        us = O.USrc(C.cast(ro.buf, C.c_void_p), None, 0, 0)
        assert L.orc_build_sampled_chain(row, C.byref(drafter), v, depth, C.byref(us), chain,
                                         dd.ctypes.data_as(C.c_void_p)) == depth
        assert [chain[i].token for i in range(depth)] == list(tok)
        assert [chain[i].path_prob for i in range(depth)] == list(pp)
        assert np.array_equal(dd, dd_ref)
        acc = _arr(C.c_int32, 64)
        alen, bonus = C.c_int32(), C.c_int32()
        assert R.ref_verify_stochastic(row, C.byref(target), v, temperature, ctx, 1, depth, tok,
                                       dd_ref.ctypes.data_as(C.c_void_p), rr, acc, C.byref(alen),
                                       C.byref(bonus)) == 0
        res = O.Accept()
        assert L.orc_verify_stochastic(row, C.byref(target), v, temperature, chain, depth,
                                       dd.ctypes.data_as(C.c_void_p), C.byref(us), C.byref(res)) == 0
        assert (res.accept_length, res.bonus) == (alen.value, bonus.value)
        assert R.ref_rng_next_u64(rr) == ro.next_u64()  # identical draw consumption
        R.ref_rng_destroy(rr)


def test_stochastic_one_hot_proposals_match():
    """chain_from_tokens proposals (no draft_dist): accept prob = p(x)."""
    R, L = O.ref(), O.orc()
    row = O.fnptr(L, "orc_test_row")
    for seed in range(40):
        v, n = 6, 3
        target = O.TestRows(seed, v, 3, 20)
        toks = [random.Random(seed).randrange(v) for _ in range(n)]
        tok = (C.c_int32 * n)(*toks)
        rr = R.ref_rng_create(seed, 9)
        ro = O.Rng(seed, 9)
        acc = _arr(C.c_int32, 8)
        alen, bonus = C.c_int32(), C.c_int32()
        ctx = (C.c_int32 * 1)(2)  # not BEGIN(1): keeps table keys distinct
        assert R.ref_verify_stochastic(row, C.byref(target), v, 1.0, ctx, 1, n, tok, None, rr, acc,
                                       C.byref(alen), C.byref(bonus)) == 0
        chain = (O.Node * n)(*[O.Node(t, i - 1, i + 1, 1.0, 1.0) for i, t in enumerate(toks)])
        us = O.USrc(C.cast(ro.buf, C.c_void_p), None, 0, 0)
        res = O.Accept()
        assert L.orc_verify_stochastic(row, C.byref(target), v, 1.0, chain, n, None, C.byref(us),
                                       C.byref(res)) == 0
        assert (res.accept_length, res.bonus) == (alen.value, bonus.value)
        R.ref_rng_destroy(rr)


# ------------------------------------------------------------- BEG-MAB
DEFAULT_ARMS = [(10, 8, 64), (6, 8, 64), (10, 8, 48), (6, 8, 48), (10, 8, 32), (6, 8, 32), (10, 8, 16), (6, 8, 16)]


@pytest.mark.parametrize("arms,thr,eps,win", [
    (DEFAULT_ARMS, [1, 2, 8, 16], 0.1, 20),
    ([(4 + i, 2, 4) for i in range(4)], [1], 0.3, 5),
    ([(10, 8, 64), (10, 8, 48), (10, 8, 32), (10, 8, 16)], [1, 2, 8, 16], 1.0, 20),
    ([(3, 2, 6), (4, 2, 6), (2, 3, 6), (5, 1, 5), (4, 1, 4)], [2, 5, 9], 0.0, 3),
])
def test_beg_mab_sequences_match(arms, thr, eps, win):
    R, L = O.ref(), O.orc()
    n = len(arms)
    dkt = (C.c_int32 * (3 * n))(*[x for a in arms for x in a])
    th = (C.c_int32 * len(thr))(*thr)
    rc = C.c_int()
    m_ref = R.ref_mab_create(dkt, n, th, len(thr), eps, win, C.byref(rc))
    assert rc.value == 0
    m_orc = C.create_string_buffer(L.orc_mab_sizeof())
    L.orc_mab_init.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_double, C.c_int]
    L.orc_mab_select.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    L.orc_mab_record.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_int]
    th_int = (C.c_int * len(thr))(*thr)
    strs = (O.Strategy * n)(*[O.Strategy(*a) for a in arms])
    assert L.orc_mab_init(m_orc, strs, n, th_int, len(thr), eps, win) == 0
    rr = R.ref_rng_create(7, 0x53454C)
    ro = O.Rng(7, 0x53454C)
    g = random.Random(5)
    for step in range(600):
        batch = g.choice([thr[0], thr[0] + 1, 3, 7, 8, 15, 16, 31, 64, 200])
        a = R.ref_mab_select(m_ref, batch, rr)
        b = L.orc_mab_select(m_orc, batch, ro.buf)
        if a < 0:
            assert b == -2 and a == -2
            continue
        assert a == b
        lens = (C.c_int32 * batch)(*[g.randrange(0, arms[a][0] + 1) for _ in range(batch)])
        elapsed = g.choice([0.5, 1.0, 2.5, g.random() + 0.01])
        assert R.ref_mab_record(m_ref, *arms[a], elapsed, lens, batch, batch) == 0
        assert L.orc_mab_record(m_orc, C.byref(strs[a]), elapsed, lens, batch) == 0
    assert R.ref_rng_next_u64(rr) == ro.next_u64()
    for i in range(n):
        med, sel, cnt, lr, la = C.c_double(), C.c_longlong(), C.c_int(), C.c_double(), C.c_double()
        R.ref_mab_stats(m_ref, i, C.byref(med), C.byref(sel), C.byref(cnt), C.byref(lr), C.byref(la))
        med2, sel2, cnt2, lr2, la2 = C.c_double(), C.c_int64(), C.c_int(), C.c_double(), C.c_double()
        assert L.orc_mab_arm_stats(m_orc, i, C.byref(med2), C.byref(sel2), C.byref(cnt2), C.byref(lr2),
                                   C.byref(la2)) == 0
        assert (med.value, sel.value, cnt.value, lr.value, la.value) == \
            (med2.value, sel2.value, cnt2.value, lr2.value, la2.value)
    R.ref_mab_destroy(m_ref)
    R.ref_rng_destroy(rr)


def test_beg_mab_config_errors_match():
    R, L = O.ref(), O.orc()
    L.orc_mab_init.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_double, C.c_int]
    cases = [([(10, 8, 64), (10, 8, 48), (10, 8, 32)], [1, 2]), ([(10, 8, 64), (10, 8, 48)], [2, 2]),
             ([(2, 1, 3)], [1]), ([(4, 2, 8)], [1])]
    for arms, thr in cases:
        n = len(arms)
        dkt = (C.c_int32 * (3 * n))(*[x for a in arms for x in a])
        rc = C.c_int()
        m = R.ref_mab_create(dkt, n, (C.c_int32 * len(thr))(*thr), len(thr), 0.1, 20, C.byref(rc))
        buf = C.create_string_buffer(L.orc_mab_sizeof())
        ok = L.orc_mab_init(buf, (O.Strategy * n)(*[O.Strategy(*a) for a in arms]), n,
                            (C.c_int * len(thr))(*thr), len(thr), 0.1, 20)
        assert (rc.value == 0) == (ok == 0)
        if m:
            R.ref_mab_destroy(m)


# -------------------------------------------------------- capture plan
@pytest.mark.parametrize("arms,thr,maxb", [
    (DEFAULT_ARMS, [1, 2, 8, 16], 32),
    ([(10, 8, 64), (10, 8, 48), (10, 8, 32), (10, 8, 16)], [1, 2, 8, 16], 32),
    ([(4, 4, 16), (4, 2, 16), (4, 4, 16), (3, 4, 8)], [1, 4], 64),
    ([(2, 2, 4)], [3], 2),  # max_batch below last threshold -> error
])
@pytest.mark.parametrize("vanilla", [0, 1])
def test_plan_captures_matches_reference(arms, thr, maxb, vanilla):
    R, L = O.ref(), O.orc()
    n = len(arms)
    dkt = (C.c_int32 * (3 * n))(*[x for a in arms for x in a])
    out6 = (C.c_int32 * (6 * 512))()
    mem = (C.c_double * 512)()
    tot = C.c_double()
    a = R.ref_plan_captures(dkt, n, (C.c_int32 * len(thr))(*thr), len(thr), maxb, vanilla, out6, mem, 512,
                            C.byref(tot))
    L.orc_plan_captures.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                    C.c_int, C.c_void_p]
    caps = (O.Capture * 512)()
    tot2 = C.c_double()
    b = L.orc_plan_captures((O.Strategy * n)(*[O.Strategy(*x) for x in arms]), n, (C.c_int * len(thr))(*thr),
                            len(thr), maxb, vanilla, caps, 512, C.byref(tot2))
    if a < 0:
        assert b < 0
        return
    assert a == b
    for i in range(a):
        c = caps[i]
        assert list(out6[6 * i:6 * i + 6]) == [c.side, c.bucket_lo, c.bucket_hi, c.tokens_to_verify, c.top_k,
                                               c.draft_depth]
        assert mem[i] == c.memory_units
    assert tot.value == tot2.value


def test_elastic_gate_and_step_latency_match():
    R, L = O.ref(), O.orc()
    L.orc_step_latency.argtypes = [C.c_int, C.c_int, C.c_void_p]
    for active in range(0, 70):
        for thr in [0, 1, 8, 32, 64]:
            a = R.ref_should_enable_sd(active, thr)
            b = L.orc_should_enable_sd(active, thr)
            assert (a < 0) == (b < 0) and (a < 0 or a == b)
    for b_ in [1, 2, 7, 32, 128]:
        for (d, k, t) in [(10, 8, 64), (4, 4, 16)]:
            assert R.ref_step_latency(b_, 1, d, k, t, 1) == L.orc_step_latency(b_, 1, C.byref(O.Strategy(d, k, t)))
        assert R.ref_step_latency(b_, 1, 0, 0, 0, 0) == L.orc_step_latency(b_, 1, None)
