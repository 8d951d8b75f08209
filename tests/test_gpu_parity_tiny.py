"""GPU engine vs CPU oracle on BASELINE config 1 (tiny Llama target + EAGLE
drafter, b=4, greedy tree SD (4,4,16)) — the parity workload.

Bit-exact bars (discrete): tree tokens/parents/depths and fp64 probs /
path_probs, accepted tokens, accepted node indices, accept lengths, bonus,
committed KV lengths, generated tokens. Checked two ways:
  * oracle-in-the-loop: the GPU's own drafter rows / verify logits are fed to
    the C restatement of build_draft_tree / verify_greedy (pinned against the
    reference in test_oracle_pinning.py) -> must reproduce the GPU tree and
    acceptance exactly, unconditionally;
  * independent: the CPU neural oracle run end to end through spec_generate
    -> same tokens (the random-init scale keeps top-1/top-2 logit margins far
    above the logit tolerance; margins are asserted).
Tolerance (floating point): logits |gpu - cpu| <= 0.05 + 0.01 |cpu|
(bf16 activations, fp32 accumulation in a different order on each side),
drafter probabilities |gpu - cpu| <= 1e-3.
"""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from paper_2511_16665_b200.engine import INITS, MODELS, Engine

pytestmark = pytest.mark.gpu

TINY = MODELS["tiny"]
INIT = INITS["tiny"]
STRAT = (4, 4, 16)
LOGIT_ATOL, LOGIT_RTOL = 0.05, 0.01


def _prompts(b=4, P=16, seed=0, V=4096):
    rng = np.random.default_rng(seed)
    return [rng.integers(2, V, P).astype(np.int32).tolist() for _ in range(b)]


@pytest.fixture(scope="module")
def omodel():
    L = O.orc()
    cfg = O.ModelCfg(TINY["vocab"], TINY["hidden"], TINY["layers"], TINY["heads"], TINY["kv_heads"],
                     TINY["head_dim"], TINY["ffn"], TINY["qkv_bias"], TINY["rope_theta"], TINY["rms_eps"], 1024)
    ini = O.InitCfg(INIT["seed"], INIT["layer_scale"], INIT["lm_gain"], INIT["lm_alt"], INIT["lm_noise"], INIT["fc_noise"],
                    int(INIT.get("drafter_lm_fp8", 0)))
    m = L.orc_model_create(C.byref(cfg), C.byref(ini), 8)
    assert m
    yield m
    L.orc_model_destroy(m)


def _oseq(m, prompt):
    L = O.orc()
    s = L.orc_seq_create(m)
    arr = (C.c_int32 * len(prompt))(*prompt)
    L.orc_seq_append.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
    assert L.orc_seq_append(s, arr, len(prompt)) == 0
    return s


def _otarget_logits(m, prompt, path=()):
    L = O.orc()
    s = _oseq(m, prompt)
    out = np.zeros(TINY["vocab"], np.float32)
    p = (C.c_int32 * max(1, len(path)))(*path)
    L.orc_target_logits_path.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    assert L.orc_target_logits_path(s, p, len(path), out.ctypes.data_as(C.c_void_p)) == 0
    L.orc_seq_destroy(s)
    return out


def _odrafter_row(m, prompt, path=()):
    L = O.orc()
    s = _oseq(m, prompt)
    probs = np.zeros(TINY["vocab"], np.float64)
    p = (C.c_int32 * max(1, len(path)))(*path)
    L.orc_drafter_row.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    assert L.orc_drafter_row(s, p, len(path), probs.ctypes.data_as(C.c_void_p), None) == 0
    L.orc_seq_destroy(s)
    return probs


def _close(gpu, cpu):
    return np.all(np.abs(gpu - cpu) <= LOGIT_ATOL + LOGIT_RTOL * np.abs(cpu))


def test_ar_logits_and_tokens_match_oracle(omodel):
    eng = Engine("tiny", max_slots=4, max_ctx=512)
    eng.set_debug(True)
    prompts = _prompts()
    eng.prefill(range(4), prompts)
    toks, _ = eng.ar_step(list(range(4)))
    lg = eng.debug_ar_logits(4)
    for i, p in enumerate(prompts):
        ref = _otarget_logits(omodel, p)
        err = np.abs(lg[i] - ref).max()
        assert _close(lg[i], ref), f"request {i}: max |dlogit| = {err}"
        srt = np.sort(ref)
        assert srt[-1] - srt[-2] > 4 * (LOGIT_ATOL + LOGIT_RTOL * abs(srt[-1])), "argmax margin too small"
        assert toks[i] == int(np.argmax(ref))
    eng.close()


def _row_cb(table, V):
    def cb(user, path, n, out):
        key = tuple(path[j] for j in range(n))
        row = table.get(key)
        if row is None:
            return -1
        C.memmove(out, row.ctypes.data, V * 8)
        return 0
    return O.ROW_FN(cb)


def _argmax_cb(table):
    def cb(user, path, n):
        key = tuple(path[j] for j in range(n))
        return table.get(key, -1)
    return O.ARGMAX_FN(cb)


def _tree_paths(tree):
    paths = []
    for n, (tok, par, _, _, _) in enumerate(tree):
        paths.append((paths[par] if par >= 0 else ()) + (tok,))
    return paths


@pytest.mark.parametrize("strategy", [STRAT, (4, 2, 8), (3, 1, 3), (5, 4, 24), (2, 8, 16)])
def test_sd_step_oracle_in_the_loop(omodel, strategy):
    """GPU tree + acceptance == C restatement fed the GPU's own rows."""
    L = O.orc()
    V = TINY["vocab"]
    eng = Engine("tiny", max_slots=4, max_ctx=512)
    eng.set_debug(True)
    prompts = _prompts(seed=3)
    eng.prefill(range(4), prompts)
    lens0 = [eng.slot_len(i) for i in range(4)]
    for step in range(3):
        r = eng.sd_step(strategy, list(range(4)))
        for i in range(4):
            exps = dict(eng.debug_expansions(i))
            cb = _row_cb(exps, V)
            out = (O.Node * strategy[2])()
            L.orc_build_draft_tree.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
            n = L.orc_build_draft_tree(C.cast(cb, C.c_void_p), None, V, C.byref(O.Strategy(*strategy)), out)
            assert n == len(r.tree[i]), (step, i)
            ref = [(out[j].token, out[j].parent, out[j].depth, out[j].prob, out[j].path_prob) for j in range(n)]
            assert ref == r.tree[i], (step, i)
            # acceptance from the GPU's verify logits
            vl = eng.debug_verify_logits(i)
            paths = _tree_paths(r.tree[i])
            table = {(): int(np.argmax(vl[0]))}
            for nd, pth in enumerate(paths):
                table[pth] = int(np.argmax(vl[1 + nd]))
            acb = _argmax_cb(table)
            res = O.Accept()
            L.orc_verify_greedy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
            assert L.orc_verify_greedy(C.cast(acb, C.c_void_p), None, out, n, C.byref(res)) == 0
            a = res.accept_length
            assert a == r.accept_len[i] and res.bonus == r.bonus[i]
            assert list(res.accepted[:a]) == r.accepted[i]
            assert list(res.nodes[:a]) == r.nodes[i]
            assert r.kv_len[i] == lens0[i] + 1 + a  # committed KV slot map: root + accepted
            lens0[i] = int(r.kv_len[i])
    eng.close()


def test_drafter_and_verify_rows_close_to_oracle(omodel):
    """Floating-point parity of the neural leaves (drafter rows, verify logits)."""
    eng = Engine("tiny", max_slots=4, max_ctx=512)
    eng.set_debug(True)
    prompts = _prompts(seed=5)
    eng.prefill(range(4), prompts)
    r = eng.sd_step(STRAT, list(range(4)))
    for i in range(4):
        exps = eng.debug_expansions(i)
        for path, row in exps[:6]:
            ref = _odrafter_row(omodel, prompts[i], path)
            # log-probabilities are logits up to a per-row constant: same tolerance class
            m = ref > 1e-6
            err = np.abs(np.log(row[m]) - np.log(ref[m]))
            assert err.max() < 2 * (LOGIT_ATOL + LOGIT_RTOL * 10), (i, path, err.max())
            assert abs(row.sum() - 1.0) < 1e-6
        vl = eng.debug_verify_logits(i)
        paths = _tree_paths(r.tree[i])
        for nd in [0, 1, 5, len(paths) - 1]:
            ref = _otarget_logits(omodel, prompts[i], paths[nd])
            assert _close(vl[1 + nd], ref), (i, nd, np.abs(vl[1 + nd] - ref).max())
        ref = _otarget_logits(omodel, prompts[i])
        assert _close(vl[0], ref)
    eng.close()


@pytest.mark.parametrize("use_graphs", [False, True])
def test_rollout_tokens_match_oracle(omodel, use_graphs):
    """End to end: GPU greedy tree SD == CPU neural spec_generate == AR."""
    L = O.orc()
    prompts = _prompts(seed=7)
    max_len = 40
    eng = Engine("tiny", max_slots=4, max_ctx=512)
    res = eng.run_rollout(prompts, [max_len] * 4, enable_sd=True, elastic_threshold=64, strategy=STRAT,
                          use_graphs=use_graphs)
    ar = eng.run_rollout(prompts, [max_len] * 4, enable_sd=False, use_graphs=use_graphs)
    L.orc_neural_spec_generate.argtypes = [C.c_void_p] * 11
    L.orc_neural_generate_ar.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]
    for i, p in enumerate(prompts):
        pa = (C.c_int32 * len(p))(*p)
        out = (C.c_int32 * 256)()
        n = C.c_int()
        acc = (C.c_int32 * 256)()
        steps = L.orc_neural_spec_generate(omodel, pa, len(p), max_len, C.byref(O.Strategy(*STRAT)), out,
                                           C.byref(n), acc, None, None, 256)
        assert steps > 0
        cpu_sd = list(out[:n.value])
        aro = (C.c_int32 * 256)()
        g = L.orc_neural_generate_ar(omodel, pa, len(p), max_len, aro)
        cpu_ar = list(aro[:g])
        assert cpu_sd == cpu_ar  # the oracle itself is lossless (spec_decode.hpp:349-350)
        assert res["tokens"][i] == cpu_sd, f"request {i}"
        assert ar["tokens"][i] == cpu_ar, f"request {i} (AR)"
    assert res["sd_steps"] > 0 and res["plain_steps"] == 0
    assert ar["plain_steps"] > 0 and ar["sd_steps"] == 0
    eng.close()


def test_fp8_drafter_lm_head_rows_and_tree_match_oracle():
    """drafter_lm_fp8 (the 7B default): the engine's e4m3 drafter LM head
    (per-row scales, kind::f8f6f4 GEMM) against the oracle's emulation of the
    same quantisation -- drafter rows within the log-prob tolerance, the tree
    bit-exact with the oracle-in-the-loop, and SD still lossless vs AR."""
    L = O.orc()
    ini8 = dict(INIT, drafter_lm_fp8=1)
    cfg = O.ModelCfg(TINY["vocab"], TINY["hidden"], TINY["layers"], TINY["heads"], TINY["kv_heads"],
                     TINY["head_dim"], TINY["ffn"], TINY["qkv_bias"], TINY["rope_theta"], TINY["rms_eps"], 1024)
    icfg = O.InitCfg(ini8["seed"], ini8["layer_scale"], ini8["lm_gain"], ini8["lm_alt"], ini8["lm_noise"],
                     ini8["fc_noise"], 1)
    m8 = L.orc_model_create(C.byref(cfg), C.byref(icfg), 8)
    assert m8
    eng = Engine("tiny", max_slots=4, max_ctx=512, init={"drafter_lm_fp8": 1})
    eng.set_debug(True)
    prompts = _prompts(seed=11)
    eng.prefill(range(4), prompts)
    r = eng.sd_step(STRAT, list(range(4)))
    for i in range(4):
        exps = eng.debug_expansions(i)
        for path, row in exps[:6]:
            ref = _odrafter_row(m8, prompts[i], path)
            msk = ref > 1e-6
            err = np.abs(np.log(row[msk]) - np.log(ref[msk]))
            assert err.max() < 2 * (LOGIT_ATOL + LOGIT_RTOL * 10), (i, path, err.max())
        table = dict(exps)

        def cb(user, path, n, out, table=table):
            row = table.get(tuple(path[j] for j in range(n)))
            if row is None:
                return -1
            C.memmove(out, row.ctypes.data, TINY["vocab"] * 8)
            return 0

        fn = O.ROW_FN(cb)
        out = (O.Node * STRAT[2])()
        L.orc_build_draft_tree.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        n = L.orc_build_draft_tree(C.cast(fn, C.c_void_p), None, TINY["vocab"], C.byref(O.Strategy(*STRAT)), out)
        assert [(out[j].token, out[j].parent, out[j].depth, out[j].prob, out[j].path_prob) for j in range(n)] == r.tree[i]
    eng.close()
    L.orc_model_destroy(m8)
