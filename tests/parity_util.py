"""Oracle-in-the-loop helpers shared by the GPU parity tests (test
infrastructure: only tests import oracle/).

check_tree_step feeds the GPU's own drafter rows (debug export of the step)
to the C restatement of build_draft_tree (spec_decode.hpp:111-197) and the
argmax of the GPU's verify logits to verify_greedy (spec_decode.hpp:245-268),
both pinned against the unmodified reference in test_oracle_pinning.py, and
asserts the GPU step's tree, acceptance and committed KV length bit for bit.
"""
import ctypes as C

import numpy as np

import oracle as O


def row_cb(table, V):
    def cb(user, path, n, out):
        row = table.get(tuple(path[j] for j in range(n)))
        if row is None:
            return -1
        C.memmove(out, row.ctypes.data, V * 8)
        return 0
    return O.ROW_FN(cb)


def argmax_cb(table):
    def cb(user, path, n):
        return table.get(tuple(path[j] for j in range(n)), -1)
    return O.ARGMAX_FN(cb)


def tree_paths(tree):
    paths = []
    for tok, par, _, _, _ in tree:
        paths.append((paths[par] if par >= 0 else ()) + (tok,))
    return paths


def check_tree_step(eng, strategy, r, i, V, kv_len_before, tag=""):
    """Asserts step result r (StepResult of eng.sd_step) for request i equals
    the oracle fed the GPU rows; returns the new committed KV length."""
    L = O.orc()
    exps = dict(eng.debug_expansions(i))
    cb = row_cb(exps, V)
    out = (O.Node * strategy[2])()
    L.orc_build_draft_tree.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    n = L.orc_build_draft_tree(C.cast(cb, C.c_void_p), None, V, C.byref(O.Strategy(*strategy)), out)
    assert n == len(r.tree[i]), (tag, i, n, len(r.tree[i]))
    ref = [(out[j].token, out[j].parent, out[j].depth, out[j].prob, out[j].path_prob) for j in range(n)]
    assert ref == r.tree[i], (tag, i)
    vl = eng.debug_verify_logits(i)
    paths = tree_paths(r.tree[i])
    table = {(): int(np.argmax(vl[0]))}
    for nd, pth in enumerate(paths):
        table[pth] = int(np.argmax(vl[1 + nd]))
    acb = argmax_cb(table)
    res = O.Accept()
    L.orc_verify_greedy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    assert L.orc_verify_greedy(C.cast(acb, C.c_void_p), None, out, n, C.byref(res)) == 0
    a = res.accept_length
    assert a == r.accept_len[i] and res.bonus == r.bonus[i], (tag, i, a, int(r.accept_len[i]))
    assert list(res.accepted[:a]) == r.accepted[i], (tag, i)
    assert list(res.nodes[:a]) == r.nodes[i], (tag, i)
    # committed KV slot map: root at L, accepted node j's KV moved to L+1+j
    assert r.kv_len[i] == kv_len_before + 1 + a, (tag, i)
    return int(r.kv_len[i])


def same_step(a, b):
    """Two StepResults of the same (engine state, strategy) are identical."""
    assert a.accept_len.tolist() == b.accept_len.tolist()
    assert a.bonus.tolist() == b.bonus.tolist()
    assert a.accepted == b.accepted and a.nodes == b.nodes
    assert a.kv_len.tolist() == b.kv_len.tolist()
    assert a.tree == b.tree


def tiny_oracle_model():
    """CPU neural oracle of the tiny (config 1) model; caller destroys it."""
    from paper_2511_16665_b200.engine import INITS, MODELS
    T, I = MODELS["tiny"], INITS["tiny"]
    L = O.orc()
    cfg = O.ModelCfg(T["vocab"], T["hidden"], T["layers"], T["heads"], T["kv_heads"], T["head_dim"], T["ffn"],
                     T["qkv_bias"], T["rope_theta"], T["rms_eps"], 1024)
    ini = O.InitCfg(I["seed"], I["layer_scale"], I["lm_gain"], I["lm_alt"], I["lm_noise"], I["fc_noise"],
                    int(I.get("drafter_lm_fp8", 0)))
    return L.orc_model_create(C.byref(cfg), C.byref(ini), 8)


def oracle_logits(m, ctx, vocab):
    """fp32 target logits of the oracle after ctx (committed tokens)."""
    L = O.orc()
    s = L.orc_seq_create(m)
    arr = (C.c_int32 * len(ctx))(*ctx)
    L.orc_seq_append.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
    assert L.orc_seq_append(s, arr, len(ctx)) == 0
    out = np.zeros(vocab, np.float32)
    L.orc_target_logits_path.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    assert L.orc_target_logits_path(s, (C.c_int32 * 1)(0), 0, out.ctypes.data_as(C.c_void_p)) == 0
    L.orc_seq_destroy(s)
    return out


def greedy_streams_agree(m, prompt, a, b, vocab, atol=0.05, rtol=0.01):
    """Two greedy token streams of the same prompt are equal, or first differ
    at a floating-point near-tie: the oracle's logits of the two candidate
    tokens at the divergence are within twice the logit tolerance (the GPU
    paths compute those logits with different reduction orders, SURVEY.md §7
    "batch invariance"). Returns (ok, divergence position or -1, margin)."""
    n = min(len(a), len(b))
    k = next((j for j in range(n) if a[j] != b[j]), None)
    if k is None:
        return True, -1, None
    lg = oracle_logits(m, list(prompt) + list(a[:k]), vocab)
    ta, tb = a[k], b[k]
    margin = abs(float(lg[ta]) - float(lg[tb]))
    tol = 2 * (atol + rtol * max(abs(float(lg[ta])), abs(float(lg[tb]))))
    return margin <= tol, k, margin
