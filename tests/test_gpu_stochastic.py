"""GPU rejection-sampling SD (K9, config 4 semantics) vs the C restatement of
build_sampled_chain / verify_stochastic (pinned to the reference in
test_oracle_pinning.py), fed the GPU's own drafter rows, the GPU's raw target
rows and the SAME RngStream uniforms. Bars: drafted chain, accept length,
bonus and uniform consumption bit-exact; KV length = root + accepted."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from paper_2511_16665_b200.engine import INITS, MODELS, Engine

pytestmark = pytest.mark.gpu

V = 4096
# config 4 at V = 152064: the Qwen2.5-32B shape truncated to 2 of its 64
# layers (the discrete rejection-sampling logic does not depend on depth;
# the full 64-layer model runs in tools/config4.py / bench configs)
MODEL_32B_TRUNC = dict(MODELS["qwen2.5-32b"], layers=2)


def _engine(model, max_slots, max_ctx):
    if model == "32b-trunc":
        return Engine(MODEL_32B_TRUNC, max_slots=max_slots, max_ctx=max_ctx, init=INITS["qwen2.5-32b"])
    return Engine(model, max_slots=max_slots, max_ctx=max_ctx)


def _uniforms(seed, stream, n):
    r = O.Rng(seed, stream)
    return [r.uniform01() for _ in range(n)]


@pytest.mark.parametrize("model,D,temperature", [("tiny", 4, 0.9), ("tiny", 3, 1.0), ("tiny", 6, 0.7),
                                                 ("32b-trunc", 4, 0.9), ("32b-trunc", 6, 0.9)])
def test_stochastic_step_oracle_in_the_loop(model, D, temperature):
    L = O.orc()
    L.orc_build_sampled_chain.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                          C.c_void_p]
    L.orc_verify_stochastic.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_void_p, C.c_int,
                                        C.c_void_p, C.c_void_p, C.c_void_p]
    eng = _engine(model, 4, 512)
    V = eng.vocab
    eng.set_debug(True)
    rng = np.random.default_rng(11)
    prompts = [rng.integers(2, V, 16).tolist() for _ in range(4)]
    eng.prefill(range(4), prompts)
    lens = [eng.slot_len(i) for i in range(4)]
    for step in range(3):
        uni = np.array([_uniforms(100 + step, 0x52515254 + i, 2 * D + 1) for i in range(4)])
        res, chains, consumed = eng.sd_step_stochastic(D, temperature, [0, 1, 2, 3], uni)
        for i in range(4):
            qrows = [row for _, row in eng.debug_expansions(i)]
            assert len(qrows) == D
            assert all(abs(r.sum() - 1.0) < 1e-9 for r in qrows)

            def draft_cb(user, path, n, out, qrows=qrows):
                C.memmove(out, qrows[n].ctypes.data, V * 8)
                return 0

            dfn = O.ROW_FN(draft_cb)
            ubuf = (C.c_double * (2 * D + 1))(*uni[i].tolist())
            us = O.USrc(None, C.cast(ubuf, O.f64p), 2 * D + 1, 0)
            nodes = (O.Node * D)()
            dd = np.zeros(D * V)
            assert L.orc_build_sampled_chain(C.cast(dfn, C.c_void_p), None, V, D, C.byref(us), nodes,
                                             dd.ctypes.data_as(C.c_void_p)) == D
            assert [nodes[j].token for j in range(D)] == chains[i], (step, i)
            rows = eng.debug_target_rows(i)
            table = {tuple(chains[i][:j]): rows[j] for j in range(D + 1)}

            def target_cb(user, path, n, out, table=table):
                row = table.get(tuple(path[j] for j in range(n)))
                if row is None:
                    return -1
                C.memmove(out, row.ctypes.data, V * 8)
                return 0

            tfn = O.ROW_FN(target_cb)
            acc = O.Accept()
            assert L.orc_verify_stochastic(C.cast(tfn, C.c_void_p), None, V, temperature, nodes, D,
                                           dd.ctypes.data_as(C.c_void_p), C.byref(us), C.byref(acc)) == 0
            a = acc.accept_length
            assert (a, acc.bonus) == (int(res.accept_len[i]), int(res.bonus[i])), (step, i)
            assert list(acc.accepted[:a]) == res.accepted[i]
            assert consumed[i] == us.cursor  # identical RngStream consumption
            assert res.kv_len[i] == lens[i] + 1 + a
            lens[i] = int(res.kv_len[i])
    eng.close()


def test_stochastic_rejects_zero_temperature():
    eng = Engine("tiny", max_slots=1, max_ctx=128)
    eng.prefill([0], [[2, 3, 4]])
    from paper_2511_16665_b200.engine import ConfigError
    with pytest.raises(ConfigError):
        eng.sd_step_stochastic(3, 0.0, [0], np.zeros((1, 7)))
    eng.close()


def test_stochastic_rollout_deterministic_and_terminates():
    """run_rollout in stochastic_linear mode (config 4 semantics): the plain
    steps sample with one draw each, SD steps consume the exact reference draw
    count; same seed -> same tokens; nothing after EOS, lengths <= max_len."""
    rng = np.random.default_rng(3)
    prompts = [rng.integers(2, V, 12).tolist() for _ in range(4)]
    outs = []
    for _ in range(2):
        eng = Engine("tiny", max_slots=4, max_ctx=512)
        r = eng.run_rollout(prompts, [40, 25, 33, 18], enable_sd=True, elastic_threshold=3, strategy=(4, 1, 4),
                            seed=9, mode="stochastic", temperature=0.9)
        outs.append(r)
        eng.close()
    assert outs[0]["tokens"] == outs[1]["tokens"]
    assert outs[0]["sd_steps"] > 0 and outs[0]["plain_steps"] > 0
    for toks, ml in zip(outs[0]["tokens"], [40, 25, 33, 18]):
        assert 1 <= len(toks) <= ml
        if 0 in toks:
            assert toks.index(0) == len(toks) - 1


def test_stochastic_first_token_marginal_is_target():
    """Losslessness (reference FirstEmittedTokenMatchesTargetEmpirically,
    spec_decode_test.cpp:357-383): the first emitted token of a rejection-
    sampling step is distributed as the tempered target row. Checked on the
    target's top tokens with 5-sigma binomial bounds."""
    D, t, n_iter = 3, 1.0, 400
    eng = Engine("tiny", max_slots=4, max_ctx=256, init=dict(lm_gain=3.0, lm_alt=0.9))
    eng.set_debug(True)
    prompt = np.random.default_rng(5).integers(2, V, 12).tolist()
    g = np.random.default_rng(123)
    counts = np.zeros(V)
    p0 = None
    for it in range(n_iter):
        eng.prefill([0, 1, 2, 3], [prompt] * 4)
        uni = g.random((4, 2 * D + 1))
        res, chains, _ = eng.sd_step_stochastic(D, t, [0, 1, 2, 3], uni)
        if p0 is None:
            p0 = eng.debug_target_rows(0)[0]  # root row (raw == tempered at t = 1)
        for i in range(4):
            first = res.accepted[i][0] if res.accept_len[i] > 0 else int(res.bonus[i])
            counts[first] += 1
    n = counts.sum()
    top = np.argsort(-p0)[:5]
    for tok in top:
        p = p0[tok]
        sigma = np.sqrt(p * (1 - p) / n)
        assert abs(counts[tok] / n - p) < 5 * sigma + 1e-3, (int(tok), counts[tok] / n, p)
    eng.close()


def _blocked_prefix(p, nthreads=256):
    """The GPU fast path's blocked prefix sums (inverse_cdf_block, stochastic.cu):
    contiguous segments per thread, segment sums exclusive-scanned in order."""
    V = len(p)
    per = (V + nthreads - 1) // nthreads
    seg = [float(np.cumsum(p[a:a + per])[-1]) if a < V else 0.0 for a in range(0, per * nthreads, per)]
    out = np.zeros(V)
    c = 0.0
    for j in range(nthreads):
        a = j * per
        cum = c
        for t in range(a, min(V, a + per)):
            cum += p[t]
            out[t] = cum
        c += seg[j]
    return out


def _ref_pick(p, u):
    """inverse_cdf_pick (token_model.hpp:83-91): sequential cumulative sum."""
    cum = 0.0
    for t in range(len(p) - 1):
        cum += p[t]
        if u < cum:
            return t
    return len(p) - 1


@pytest.mark.parametrize("model", ["tiny", "32b-trunc"])
def test_inverse_cdf_exact_at_cdf_boundaries(model):
    """The chain draw equals the reference's sequential inverse CDF even when
    u sits exactly on, or within rounding of, a CDF boundary (the blocked scan
    and the sequential sum round differently there)."""
    eng = _engine(model, 1, 256)
    V = eng.vocab
    eng.set_debug(True)
    prompt = np.random.default_rng(7).integers(2, V, 12).tolist()
    eng.prefill([0], [prompt])
    eng.sd_step_stochastic(1, 1.0, [0], np.full((1, 3), 0.5))
    q0 = eng.debug_expansions(0)[0][1]  # drafter root row (fp64) the chain draw used
    seq = np.cumsum(q0)  # numpy accumulate: the reference's sequential order
    blk = _blocked_prefix(q0)
    us = []
    top = np.argsort(-q0)[:6]
    for t in top:  # exact boundaries of the heaviest tokens and their neighbours
        us += [float(seq[t]), float(np.nextafter(seq[t], 0.0)), float(np.nextafter(seq[t], 1.0))]
    diff = np.nonzero(seq[:-1] != blk[:-1])[0]
    for t in diff[:6]:  # boundaries where the blocked and sequential sums disagree
        lo, hi = sorted((float(seq[t]), float(blk[t])))
        us += [lo, hi, (lo + hi) / 2]
    us = [u for u in us if 0.0 <= u < 1.0]
    assert us
    for u in us:
        eng.release(0)
        eng.prefill([0], [prompt])
        _, chains, _ = eng.sd_step_stochastic(1, 1.0, [0], np.array([[u, 0.5, 0.5]]))
        assert chains[0][0] == _ref_pick(q0, u), (u, chains[0][0])
    eng.close()
