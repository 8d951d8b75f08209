"""CPU tests of the C-ABI boundary (no GPU compute): the library loads, exports
every symbol include/tlt_b200.h declares, and its host-side strategy selection
(BEG-MAB), RngStream and capture plan are bit-identical to the reference."""
import ctypes as C
import os
import random
import re

import numpy as np
import pytest

import oracle as O
from paper_2511_16665_b200 import _lib
from paper_2511_16665_b200.engine import ConfigError, Mab, RoutingError, Rng, plan_captures

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "tlt_b200.h")).read()
    return sorted(set(re.findall(r"TLT_API\s+[\w\s\*]+?\b(tlt_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = _declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert L.tlt_version().startswith(b"tlt_b200")


def test_errors_map_to_reference_exceptions():
    with pytest.raises(ConfigError):
        Mab([(2, 1, 3)], [1])  # capacity: chain of depth 2 holds 2 nodes (spec_decode.hpp:40)
    with pytest.raises(ConfigError):
        Mab([(10, 8, 64), (10, 8, 48)], [1])  # group/threshold mismatch (beg_mab.hpp:99)
    m = Mab([(10, 8, 64), (10, 8, 48)], [2, 8])
    with pytest.raises(RoutingError):
        m.select(1, Rng(1, 0))  # below smallest bucket (beg_mab.hpp:141-143)
    with pytest.raises(ConfigError):
        m.record((10, 8, 64), 0.0, [1])  # elapsed must be > 0
    with pytest.raises(ConfigError):
        m.record((9, 9, 9), 1.0, [1])  # unknown strategy


needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference bridge not built")


@needs_ref
@pytest.mark.parametrize("seed,stream", [(0, 0), (42, 0x53454C), (7, 0x52515254 + 5)])
def test_product_rng_matches_reference(seed, stream):
    R = O.ref()
    r = R.ref_rng_create(seed, stream)
    p = Rng(seed, stream)
    for _ in range(400):
        assert R.ref_rng_next_u64(r) == p.next_u64()
    rf, pf = R.ref_rng_fork(r, 99), p.fork(99)
    for _ in range(50):
        assert R.ref_rng_uniform01(rf) == pf.uniform01()
    R.ref_rng_destroy(r)
    R.ref_rng_destroy(rf)


DEFAULT_ARMS = [(10, 8, 64), (6, 8, 64), (10, 8, 48), (6, 8, 48), (10, 8, 32), (6, 8, 32), (10, 8, 16), (6, 8, 16)]


@needs_ref
@pytest.mark.parametrize("eps", [0.0, 0.1, 1.0])
def test_product_mab_matches_reference(eps):
    R = O.ref()
    n = len(DEFAULT_ARMS)
    dkt = (C.c_int32 * (3 * n))(*[x for a in DEFAULT_ARMS for x in a])
    thr = [1, 2, 8, 16]
    rc = C.c_int()
    mref = R.ref_mab_create(dkt, n, (C.c_int32 * 4)(*thr), 4, eps, 20, C.byref(rc))
    assert rc.value == 0
    mp = Mab(DEFAULT_ARMS, thr, eps, 20)
    rr = R.ref_rng_create(3, 0x53454C)
    rp = Rng(3, 0x53454C)
    g = random.Random(11)
    for _ in range(500):
        batch = g.choice([1, 2, 5, 7, 8, 12, 15, 16, 31])
        a = R.ref_mab_select(mref, batch, rr)
        b, s = mp.select(batch, rp)
        assert a == b and s == DEFAULT_ARMS[a]
        lens = [g.randrange(0, 11) for _ in range(batch)]
        el = g.random() * 5 + 0.01
        assert R.ref_mab_record(mref, *s, el, (C.c_int32 * batch)(*lens), batch, batch) == 0
        mp.record(s, el, lens)
    for i in range(n):
        med, sel, cnt = C.c_double(), C.c_longlong(), C.c_int()
        lr, la = C.c_double(), C.c_double()
        R.ref_mab_stats(mref, i, C.byref(med), C.byref(sel), C.byref(cnt), C.byref(lr), C.byref(la))
        assert mp.arm_stats(i) == (med.value, sel.value, cnt.value)
    R.ref_mab_destroy(mref)
    R.ref_rng_destroy(rr)


@needs_ref
@pytest.mark.parametrize("vanilla", [False, True])
def test_product_plan_captures_matches_reference(vanilla):
    R = O.ref()
    n = len(DEFAULT_ARMS)
    dkt = (C.c_int32 * (3 * n))(*[x for a in DEFAULT_ARMS for x in a])
    out6 = (C.c_int32 * (6 * 256))()
    mem = (C.c_double * 256)()
    tot = C.c_double()
    k = R.ref_plan_captures(dkt, n, (C.c_int32 * 4)(1, 2, 8, 16), 4, 32, int(vanilla), out6, mem, 256,
                            C.byref(tot))
    entries, total = plan_captures(DEFAULT_ARMS, [1, 2, 8, 16], 32, vanilla)
    assert k == len(entries) and total == tot.value
    for i, e in enumerate(entries):
        assert list(e[:6]) == list(out6[6 * i:6 * i + 6]) and e[6] == mem[i]
    if not vanilla:
        # the bucketed plan of the reference simulator: 4 TARGET + 8 DRAFT graphs
        assert sum(1 for e in entries if e[0] == 0) == 4


def test_mab_merge_of_foreign_records_is_order_deterministic():
    """C1 merge semantics: applying the same records in rank order yields
    identical replicas (tests/test_multiproc_stats.py runs it over gloo)."""
    a = Mab(DEFAULT_ARMS, [1, 2, 8, 16])
    b = Mab(DEFAULT_ARMS, [1, 2, 8, 16])
    recs = [(3, 120.5, 4.25), (0, 80.0, 3.0), (3, 99.0, 2.5)]
    for arm, r, ab in recs:
        a.apply_record(arm, r, ab)
        b.apply_record(arm, r, ab)
    for i in range(len(DEFAULT_ARMS)):
        assert a.arm_stats(i) == b.arm_stats(i)
    assert a.arm_stats(3)[2] == 2 and a.arm_stats(3)[0] == pytest.approx((120.5 + 99.0) / 2)


@needs_ref
def test_product_step_latency_matches_reference():
    """tlt_step_latency (the parity_elapsed clock) == reference step_latency
    (cost_model.hpp:38-48) with the default CostModelParams."""
    from paper_2511_16665_b200.engine import step_latency
    R = O.ref()
    R.ref_step_latency.argtypes = [C.c_int] * 6
    for batch in [1, 2, 7, 16, 31, 64, 377, 1000]:
        assert step_latency(batch, 1) == R.ref_step_latency(batch, 1, 0, 0, 0, 0)
        for s in DEFAULT_ARMS + [(4, 4, 16), (2, 1, 2)]:
            assert step_latency(batch, s[2], s) == R.ref_step_latency(batch, s[2], *s, 1)


def test_step_latency_cost_validation():
    from paper_2511_16665_b200.engine import ConfigError, CostModel, step_latency
    c = CostModel(0.5, 2.0, 1.0, 1.0, 100.0, 0.25)
    assert step_latency(8, 1, None, c) == 0.5 + 2.0
    assert step_latency(100, 16, (4, 4, 16), c) == 0.5 + 16.0 + 4 * 0.25
    with pytest.raises(ConfigError, match="cost_model.mem_bw"):
        step_latency(1, 1, None, CostModel(0.5, 2.0, -1.0, 1.0, 100.0, 0.25))
    with pytest.raises(ConfigError, match="batch"):
        step_latency(0, 1)
