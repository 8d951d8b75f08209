"""Model-free n-gram fallback drafter.

Host index (tlt_ngram_*, csrc/host_select.h `Ngram`) pinned bit-for-bit
against the UNMODIFIED reference NgramIndex / ngram_insert / ngram_draft
(ngram.hpp:13-103) and NgramTracker::extend (rollout.hpp:103-120) through
oracle/_ref; the GPU chain verify (tlt_sd_step_chain) is checked against the
same engine's greedy plain decode, which greedy SD must reproduce token for
token (spec_decode.hpp:348-351 "token-identical to greedy autoregressive").
"""
import ctypes as C
import random

import numpy as np
import pytest

import oracle as O
from paper_2511_16665_b200.engine import ConfigError, Engine, Ngram


def _ref_lib():
    R = O.ref()
    R.ref_ngram_create.restype = C.c_void_p
    R.ref_ngram_destroy.argtypes = [C.c_void_p]
    R.ref_ngram_insert.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_longlong]
    R.ref_ngram_extend.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_longlong]
    R.ref_ngram_draft.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]
    R.ref_ngram_size.argtypes = [C.c_void_p]
    R.ref_ngram_size.restype = C.c_longlong
    return R


def _a(x):
    return np.ascontiguousarray(np.asarray(x, np.int32))


def _ref_draft(R, h, ctx, depth):
    c = _a(ctx)
    out = np.zeros(max(depth, 1) + 64, np.int32)
    n = R.ref_ngram_draft(h, c.ctypes.data, len(c), depth, out.ctypes.data)
    return n, out[:max(n, 0)].tolist()


@pytest.mark.skipif(not O.ref_available(), reason="reference bridge not built")
@pytest.mark.parametrize("seed,n,cont,vocab", [(0, 1, 1, 3), (1, 2, 8, 5), (2, 3, 4, 4), (3, 2, 3, 50)])
def test_ngram_index_matches_reference(seed, n, cont, vocab):
    """Random insert/extend/draft sequences over a small vocabulary (many
    frequency and recency ties), every draft compared with the reference."""
    R = _ref_lib()
    rnd = random.Random(seed)
    h = R.ref_ngram_create(n, cont)
    g = Ngram(n, cont)
    stream = []
    try:
        for step in range(60):
            op = rnd.random()
            if op < 0.35:
                resp = [rnd.randrange(vocab) for _ in range(rnd.randrange(0, 20))]
                R.ref_ngram_insert(h, _a(resp).ctypes.data, len(resp), step)
                g.insert(resp, step)
            else:
                stream += [rnd.randrange(vocab) for _ in range(rnd.randrange(1, 6))]
                R.ref_ngram_extend(h, _a(stream).ctypes.data, len(stream), step)
                g.extend(stream, step)
            assert g.size() == R.ref_ngram_size(h)
            for _ in range(4):
                ctx = [rnd.randrange(vocab) for _ in range(rnd.randrange(0, 6))]
                if rnd.random() < 0.5 and stream:
                    ctx = stream[-rnd.randrange(1, len(stream) + 1):]
                depth = rnd.randrange(1, 10)
                rn, rtok = _ref_draft(R, h, ctx, depth)
                assert rn >= 0
                assert g.draft(ctx, depth) == rtok
    finally:
        R.ref_ngram_destroy(h)


def test_ngram_tiebreaks_and_errors():
    g = Ngram(2, 3)
    g.insert([1, 2, 3, 4, 5], step_id=1)  # (1,2)->[3,4,5]
    g.insert([1, 2, 9, 9], step_id=1)     # (1,2)->[9,9]  same freq, same step, larger
    assert g.draft([7, 1, 2], 8) == [3, 4, 5]
    assert g.draft([1, 2], 2) == [3, 4]
    g.insert([1, 2, 9, 9], step_id=2)     # freq 2 wins
    assert g.draft([1, 2], 8) == [9, 9]
    assert g.draft([5], 3) == []          # context shorter than n
    assert g.draft([4, 4], 3) == []       # unknown key
    with pytest.raises(ConfigError):
        g.draft([1, 2], 0)
    with pytest.raises(ConfigError):
        Ngram(0, 2)
    with pytest.raises(ConfigError):
        Ngram(2, 0)


@pytest.mark.gpu
def test_gpu_chain_verify_matches_greedy_decode():
    """n-gram chains verified on the GPU emit exactly the greedy plain-decode
    stream; a chain equal to that stream is accepted in full; a wrong first
    token accepts nothing and emits the argmax as the bonus; KV lengths track."""
    V = 4096
    rng = np.random.default_rng(3)
    prompts = [rng.integers(2, V, 16).tolist() for _ in range(3)]
    steps = 24
    ar = Engine("tiny", max_slots=3, max_ctx=512, device=0)
    ar.prefill(range(3), prompts)
    ref = [[] for _ in range(3)]
    for _ in range(steps * 3):
        toks, _ = ar.ar_step([0, 1, 2])
        for i in range(3):
            ref[i].append(int(toks[i]))
    ar.close()

    D = 4
    eng = Engine("tiny", max_slots=3, max_ctx=512, device=0)
    eng.prefill(range(3), prompts)
    out = [[] for _ in range(3)]
    trackers = [Ngram(2, D) for _ in range(3)]
    perfect = wrong = 0
    for step in range(steps):
        chains = []
        for i in range(3):
            ctx = prompts[i] + out[i]
            mode = (step + i) % 3
            if mode == 0:       # oracle-perfect chain: the next D greedy tokens
                c = ref[i][len(out[i]):len(out[i]) + D]
            elif mode == 1:     # wrong first token
                c = [(ref[i][len(out[i])] + 1) % V, 5, 6][:D]
            else:               # the reference n-gram drafter over the request stream
                trackers[i].extend(ctx, step)
                c = trackers[i].draft(ctx, D)
            chains.append(c)
        kv0 = [len(prompts[i]) - 1 + len(out[i]) for i in range(3)]
        r = eng.sd_step_chain(D, [0, 1, 2], chains)
        for i in range(3):
            a = int(r.accept_len[i])
            emitted = r.accepted[i] + [int(r.bonus[i])]
            mode = (step + i) % 3
            if mode == 0 and len(chains[i]) == D:
                assert a == D
                perfect += 1
            if mode == 1:
                assert a == 0
                wrong += 1
            assert r.accepted[i] == chains[i][:a]
            assert r.nodes[i] == list(range(a))
            assert int(r.kv_len[i]) == kv0[i] + 1 + a
            out[i] += emitted
    for i in range(3):
        n = min(len(out[i]), len(ref[i]))
        assert n >= steps
        assert out[i][:n] == ref[i][:n]
    assert perfect > 0 and wrong > 0
    # the EAGLE path still works after chain steps (drafter catch-up)
    r = eng.sd_step((4, 4, 16), [0, 1, 2])
    for i in range(3):
        emitted = r.accepted[i] + [int(r.bonus[i])]
        pos = len(out[i])
        assert emitted == ref[i][pos:pos + len(emitted)]
    with pytest.raises(ConfigError):
        eng.sd_step_chain(D, [0], [[1, 2, 3, 4, 5]])
    eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("D", [3, 8])
def test_gpu_rollout_ngram_branch_is_lossless(D):
    """tlt_run_rollout with a stale drafter (rollout.hpp:142-144) drafts with
    the per-request n-gram tracker (rollout.hpp:212-216) and must emit the
    same greedy stream as plain decode; repetitive greedy streams of the
    random-init model give the tracker real acceptances."""
    V = 4096
    rng = np.random.default_rng(11)
    prompts = [rng.integers(2, V, 12).tolist() for _ in range(4)]
    max_lens = [96, 64, 80, 48]
    eng = Engine("tiny", max_slots=4, max_ctx=512, device=0)
    ng = eng.run_rollout(prompts, max_lens, enable_sd=True, elastic_threshold=64, strategy=(D, 1, D),
                         drafter_stale=True, ngram_n=2, ngram_continuation_len=8, target_step_id=3)
    ar = eng.run_rollout(prompts, max_lens, enable_sd=False)
    eng.close()
    # lossless: identical streams, or streams that part at a floating-point
    # near-tie of the target (oracle logits of both candidates within tolerance)
    from parity_util import greedy_streams_agree, tiny_oracle_model
    m = tiny_oracle_model()
    try:
        for p, a, b in zip(prompts, ng["tokens"], ar["tokens"]):
            ok, k, margin = greedy_streams_agree(m, p, a, b, V)
            assert ok, (k, margin)
    finally:
        O.orc().orc_model_destroy(m)
    assert ng["sd_steps"] > 0 and ng["plain_steps"] == 0
    if ng["tokens"] == ar["tokens"]:
        assert ng["emitted_total"] == sum(len(t) for t in ar["tokens"])
    assert ng["accepted_total"] > 0
    assert ng["sd_steps"] <= ar["plain_steps"]
    assert ng["verify_events"] >= ng["emitted_total"] - ng["accepted_total"]


def test_rollout_cfg_ngram_fields():
    """The ctypes mirror carries the n-gram fields in the C struct's order
    (offsets are checked against the compiled header in test_abi_layout.py)."""
    import paper_2511_16665_b200.engine as E
    names = [f[0] for f in E.RolloutCfg._fields_]
    i = names.index("drafter_stale")
    assert names[i:i + 4] == ["drafter_stale", "ngram_n", "ngram_continuation_len", "target_step_id"]


@pytest.mark.gpu
@pytest.mark.parametrize("D,temperature,scale", [(4, 0.9, 1.0), (6, 0.7, 0.02), (3, 1.0, 0.2)])
def test_gpu_chain_stochastic_oracle_in_the_loop(D, temperature, scale):
    """Stochastic n-gram branch: verify_stochastic with empty draft_dist (q
    one-hot, spec_decode.hpp:282,296-298) on the GPU vs the C restatement
    (pinned to the reference) fed the GPU's raw target rows and the SAME
    uniforms. Bars: accept length, accepted tokens, bonus and uniform
    consumption bit-exact; KV length = root + accepted. `scale` < 1 shrinks
    the uniforms so drafted tokens are also accepted."""
    L = O.orc()
    L.orc_verify_stochastic.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_void_p, C.c_int,
                                        C.c_void_p, C.c_void_p, C.c_void_p]
    V = 4096
    eng = Engine("tiny", max_slots=4, max_ctx=512, device=0)
    eng.set_debug(True)
    rng = np.random.default_rng(5)
    prompts = [rng.integers(2, V, 16).tolist() for _ in range(4)]
    eng.prefill(range(4), prompts)
    ctxs = [list(p) for p in prompts]
    trackers = [Ngram(1, D) for _ in range(4)]
    lens = [eng.slot_len(i) for i in range(4)]
    accepted_any = 0
    for step in range(8):
        # greedy continuation of every context from a twin engine (likely-accepted chains)
        twin = Engine("tiny", max_slots=4, max_ctx=512, device=0)
        twin.prefill(range(4), ctxs)
        greedy = [[] for _ in range(4)]
        for _ in range(D):
            toks, _ = twin.ar_step([0, 1, 2, 3])
            for i in range(4):
                greedy[i].append(int(toks[i]))
        twin.close()
        chains = []
        for i in range(4):
            mode = (step + i) % 4
            if mode == 0:
                c = []
            elif mode == 1:
                c = rng.integers(2, V, D).tolist()
            elif mode == 3:
                c = greedy[i]
            else:
                trackers[i].extend(ctxs[i], step)
                c = trackers[i].draft(ctxs[i], D)
            chains.append(c)
        uni = np.array([[u * scale for u in _uniforms_o(700 + step, 0x52515254 + i, D + 1)] for i in range(4)])
        res, consumed = eng.sd_step_chain_stochastic(D, temperature, [0, 1, 2, 3], chains, uni)
        for i in range(4):
            n = len(chains[i])
            rows = eng.debug_target_rows(i, max_rows=D + 1)
            table = {tuple(chains[i][:j]): rows[j] for j in range(n + 1)}

            def target_cb(user, path, k, out, table=table):
                row = table.get(tuple(path[j] for j in range(k)))
                if row is None:
                    return -1
                C.memmove(out, row.ctypes.data, V * 8)
                return 0

            tfn = O.ROW_FN(target_cb)
            ubuf = (C.c_double * (D + 1))(*uni[i].tolist())
            us = O.USrc(None, C.cast(ubuf, O.f64p), D + 1, 0)
            nodes = (O.Node * max(n, 1))()
            for j, t in enumerate(chains[i]):
                nodes[j].token, nodes[j].parent, nodes[j].depth = t, j - 1, j + 1
                nodes[j].prob = nodes[j].path_prob = 1.0
            acc = O.Accept()
            assert L.orc_verify_stochastic(C.cast(tfn, C.c_void_p), None, V, temperature, nodes, n, None,
                                           C.byref(us), C.byref(acc)) == 0
            a = acc.accept_length
            assert (a, acc.bonus) == (int(res.accept_len[i]), int(res.bonus[i])), (step, i)
            assert list(acc.accepted[:a]) == res.accepted[i] == chains[i][:a]
            assert consumed[i] == us.cursor
            assert int(res.kv_len[i]) == lens[i] + 1 + a
            lens[i] = int(res.kv_len[i])
            ctxs[i] += res.accepted[i] + [int(res.bonus[i])]
            accepted_any += a
    if scale < 0.1:
        assert accepted_any > 0
    eng.close()


def _uniforms_o(seed, stream, n):
    r = O.Rng(seed, stream)
    return [r.uniform01() for _ in range(n)]


@pytest.mark.gpu
def test_gpu_rollout_ngram_stochastic_deterministic():
    """Stochastic rollout through the n-gram branch: seeded, reproducible,
    terminates at max_len/EOS, all steps SD (batch below the gate)."""
    V = 4096
    rng = np.random.default_rng(17)
    prompts = [rng.integers(2, V, 10).tolist() for _ in range(3)]
    max_lens = [40, 24, 33]
    eng = Engine("tiny", max_slots=3, max_ctx=512, device=0)
    kw = dict(enable_sd=True, elastic_threshold=64, strategy=(4, 1, 4), mode="stochastic", temperature=0.9,
              drafter_stale=True, ngram_n=1, ngram_continuation_len=4, seed=9)
    r1 = eng.run_rollout(prompts, max_lens, **kw)
    r2 = eng.run_rollout(prompts, max_lens, **kw)
    eng.close()
    assert r1["tokens"] == r2["tokens"]
    assert r1["plain_steps"] == 0 and r1["sd_steps"] > 0
    for t, m in zip(r1["tokens"], max_lens):
        assert 1 <= len(t) <= m
        assert len(t) == m or t[-1] == 0


@pytest.mark.gpu
def test_gpu_chain_verify_7b_shape_lossless():
    """Qwen2.5-7B shape (V=152064, 28 layers): greedy chain verification of
    perfect / wrong / partially right chains reproduces plain decode."""
    rng = np.random.default_rng(21)
    prompts = [rng.integers(2, 152064, 40).tolist() for _ in range(2)]
    D, steps = 5, 6
    eng = Engine("qwen2.5-7b", max_slots=2, max_ctx=256, device=0)
    eng.prefill([0, 1], prompts)
    ref = [[], []]
    for _ in range(steps * (D + 1)):
        toks, _ = eng.ar_step([0, 1])
        for i in range(2):
            ref[i].append(int(toks[i]))
    eng.close()
    eng = Engine("qwen2.5-7b", max_slots=2, max_ctx=256, device=0)
    eng.prefill([0, 1], prompts)
    out = [[], []]
    for step in range(steps):
        chains = []
        for i in range(2):
            nxt = ref[i][len(out[i]):len(out[i]) + D]
            mode = (step + i) % 3
            if mode == 1:
                nxt = nxt[:2] + [(nxt[2] + 7) % 152064] + nxt[3:]  # wrong third token
            elif mode == 2:
                nxt = [(nxt[0] + 1) % 152064]
            chains.append(nxt)
        r = eng.sd_step_chain(D, [0, 1], chains)
        for i in range(2):
            a = int(r.accept_len[i])
            mode = (step + i) % 3
            assert a == {0: D, 1: 2, 2: 0}[mode], (step, i, a)
            out[i] += r.accepted[i] + [int(r.bonus[i])]
    eng.close()
    for i in range(2):
        assert out[i] == ref[i][:len(out[i])]
