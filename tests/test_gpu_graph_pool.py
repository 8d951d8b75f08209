"""CUDA-graph pool from plan_captures (reference
capture_plan.hpp:87-155, paper Table 3).

* the bucketed plan captures one fused step graph per (bucket, strategy) of
  the plan (default arms: 8) and the vanilla plan one per strategy x bucket
  (32); both report their real device bytes and build time;
* a BEG-MAB rollout over the pre-built pool replays only pooled graphs (no
  capture on demand) and stays lossless (== plain greedy decode);
* a step padded to its bucket's largest batch gives the same tokens and
  acceptance as the exact-batch step (padding requests inert).
"""
import numpy as np
import pytest

import oracle as O

from paper_2511_16665_b200.engine import Engine, Mab

pytestmark = pytest.mark.gpu
ARMS = [(10, 8, 64), (6, 8, 64), (10, 8, 48), (6, 8, 48), (10, 8, 32), (6, 8, 32), (10, 8, 16), (6, 8, 16)]
THR = [1, 2, 8, 16]
V = 4096


def test_bucketed_vs_vanilla_pool_sizes():
    eng = Engine("tiny", max_slots=32, max_ctx=512)
    b = eng.graph_pool_build(ARMS, THR, 32)
    v = eng.graph_pool_build(ARMS, THR, 32, vanilla=True)
    assert b["plan_entries"] == 12 and v["plan_entries"] == 64
    ar = [1, 2, 4, 8, 16, 24, 32]
    assert b["graphs"] == 8 + len(ar)
    assert v["graphs"] + v["skipped"] == 32 + len(ar)
    assert v["graphs"] > b["graphs"]
    print(f"bucketed: {b}\nvanilla: {v}")
    eng.close()


def test_mab_rollout_replays_only_pooled_graphs_and_is_lossless():
    rng = np.random.default_rng(9)
    n = 12
    prompts = [rng.integers(2, V, 10).tolist() for _ in range(n)]
    max_lens = [int(x) for x in rng.integers(8, 90, n)]
    eng = Engine("tiny", max_slots=32, max_ctx=512)
    st = eng.graph_pool_build(ARMS, THR, 32)
    sd = eng.run_rollout(prompts, max_lens, enable_sd=True, elastic_threshold=32, mab=Mab(ARMS, THR, 0.1, 20),
                         seed=1)
    after = eng.graph_pool_stats()
    assert after["live_graphs"] == st["graphs"], (st, after)  # nothing captured on demand
    ar = eng.run_rollout(prompts, max_lens, enable_sd=False)
    assert eng.graph_pool_stats()["live_graphs"] == st["graphs"]
    from parity_util import greedy_streams_agree, tiny_oracle_model
    m = tiny_oracle_model()
    try:
        for p, a, b in zip(prompts, sd["tokens"], ar["tokens"]):
            ok, k, margin = greedy_streams_agree(m, p, a, b, V)
            assert ok, (k, margin)
    finally:
        O.orc().orc_model_destroy(m)
    assert sd["sd_steps"] > 0
    # batches seen: padded into their buckets
    assert {m["batch_size"] for m in sd["trace"]} - {1, 2, 4, 8, 16, 24, 32}
    eng.close()


@pytest.mark.parametrize("b,strategy", [(5, (6, 8, 48)), (3, (10, 8, 48)), (11, (6, 8, 32)), (20, (6, 8, 16))])
def test_padded_step_equals_exact_step(b, strategy):
    """The padded step emits the same tokens as the exact-batch step. (Trees
    and acceptance may differ where drafter probabilities nearly tie: the
    padded GEMMs run a different tile / split-K plan, so logits differ in the
    last bits — SURVEY.md §7 "batch invariance"; the padded step itself is
    checked bit for bit against the oracle fed its own rows in
    test_gpu_parity_graphs.py.) The first step, from identical state, and
    every plain-decode step must agree exactly."""
    rng = np.random.default_rng(b)
    prompts = [rng.integers(2, V, 14).tolist() for _ in range(b)]
    slots = list(range(b))
    streams, firsts = [], []
    for pooled in (False, True):
        eng = Engine("tiny", max_slots=32, max_ctx=512)
        if pooled:
            eng.graph_pool_build(ARMS, THR, 32)
        eng.prefill(slots, prompts)
        out = [[] for _ in range(b)]
        for step in range(3):
            r = eng.sd_step(strategy, slots)
            if step == 0:
                firsts.append((r.accept_len.tolist(), r.bonus.tolist(), r.accepted, r.kv_len.tolist()))
            for i in range(b):
                out[i] += r.accepted[i] + [int(r.bonus[i])]
            toks, _ = eng.ar_step(slots)
            for i in range(b):
                out[i].append(int(toks[i]))
        streams.append(out)
        eng.close()
    assert firsts[0] == firsts[1]
    from parity_util import greedy_streams_agree, tiny_oracle_model
    m = tiny_oracle_model()
    try:
        for p, a, c in zip(prompts, *streams):
            n = min(len(a), len(c))
            ok, k, margin = greedy_streams_agree(m, p, a[:n], c[:n], V)
            assert ok, (k, margin)
    finally:
        O.orc().orc_model_destroy(m)
