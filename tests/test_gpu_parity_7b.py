"""Discrete parity at the BASELINE config-2 shape (Qwen2.5-7B-shaped target,
V = 152064, random-init weights): the GPU tree (tokens, parents, depths, fp64
probs / path_probs), accepted tokens / node indices / accept lengths / bonus
and the committed KV slot map must equal the C restatement of
build_draft_tree / verify_greedy (pinned against the reference in
test_oracle_pinning.py) fed the GPU's own drafter rows and verify logits.
Exercises the full-size kernels: CTA-pair and split-K GEMMs, hd=128 tree and
decode attention over several 256-key splits, V=152064 top-k / argmax."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from paper_2511_16665_b200.engine import Engine
from test_gpu_parity_tiny import _argmax_cb, _row_cb, _tree_paths

pytestmark = pytest.mark.gpu
V = 152064


@pytest.mark.parametrize("strategy,b,P", [((4, 8, 16), 2, 300), ((3, 2, 6), 3, 600)])
def test_7b_sd_step_oracle_in_the_loop(strategy, b, P):
    L = O.orc()
    eng = Engine("qwen2.5-7b", max_slots=b, max_ctx=P + 64)
    eng.set_debug(True)
    rng = np.random.default_rng(5)
    prompts = [rng.integers(2, V, P).tolist() for _ in range(b)]
    eng.prefill(range(b), prompts)
    lens0 = [eng.slot_len(i) for i in range(b)]
    for step in range(2):
        r = eng.sd_step(strategy, list(range(b)))
        for i in range(b):
            exps = dict(eng.debug_expansions(i))
            cb = _row_cb(exps, V)
            out = (O.Node * strategy[2])()
            L.orc_build_draft_tree.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
            n = L.orc_build_draft_tree(C.cast(cb, C.c_void_p), None, V, C.byref(O.Strategy(*strategy)), out)
            ref = [(out[j].token, out[j].parent, out[j].depth, out[j].prob, out[j].path_prob) for j in range(n)]
            assert ref == r.tree[i], (step, i)
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
            assert a == r.accept_len[i] and res.bonus == r.bonus[i], (step, i)
            assert list(res.accepted[:a]) == r.accepted[i]
            assert list(res.nodes[:a]) == r.nodes[i]
            assert r.kv_len[i] == lens0[i] + 1 + a
            lens0[i] = int(r.kv_len[i])
    eng.close()
