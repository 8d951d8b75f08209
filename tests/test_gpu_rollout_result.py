"""Full RolloutResult and deterministic elapsed.

The GPU rollout (tlt_run_rollout, tiny config 1 model, BEG-MAB over the
reference's default arms, parity_elapsed = 1) is replayed step by step
through the UNMODIFIED reference's beg_select / beg_record / step_latency
(oracle/_ref, rollout.hpp:130-276 control flow restated in this test) fed the
GPU's own per-step accept lengths (oracle-in-the-loop; the lengths
themselves are pinned by the tree/verify parity tests). Bit-exact bars:
  * every step's batch size, SD flag, strategy (arm), elapsed;
  * total_time, finish_time per request, accept_at_least, counters;
  * generated tokens == the CPU neural oracle's plain greedy decode
    (lossless, spec_decode.hpp:349-350), cut at EOS / max_len — up to a
    floating-point near-tie of the target logits (parity_util).
"""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from paper_2511_16665_b200.engine import INITS, MODELS, CostModel, Engine, Mab

pytestmark = pytest.mark.gpu

TINY, INIT = MODELS["tiny"], INITS["tiny"]
ARMS = [(10, 8, 64), (6, 8, 64), (10, 8, 48), (6, 8, 48), (10, 8, 32), (6, 8, 32), (10, 8, 16), (6, 8, 16)]
THR = [1, 2, 8, 16]


@pytest.fixture(scope="module")
def omodel():
    L = O.orc()
    cfg = O.ModelCfg(TINY["vocab"], TINY["hidden"], TINY["layers"], TINY["heads"], TINY["kv_heads"],
                     TINY["head_dim"], TINY["ffn"], TINY["qkv_bias"], TINY["rope_theta"], TINY["rms_eps"], 1024)
    ini = O.InitCfg(INIT["seed"], INIT["layer_scale"], INIT["lm_gain"], INIT["lm_alt"], INIT["lm_noise"],
                    INIT["fc_noise"], int(INIT.get("drafter_lm_fp8", 0)))
    m = L.orc_model_create(C.byref(cfg), C.byref(ini), 8)
    assert m
    yield m
    L.orc_model_destroy(m)


def _oracle_ar(m, prompt, max_len):
    L = O.orc()
    L.orc_neural_generate_ar.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]
    out = (C.c_int32 * (max_len + 8))()
    g = L.orc_neural_generate_ar(m, (C.c_int32 * len(prompt))(*prompt), len(prompt), max_len, out)
    return list(out[:g])


class _RefMab:
    """The unmodified reference BEG-MAB (beg_mab.hpp) through oracle/_ref."""

    def __init__(self, eps, window):
        self.R = O.ref()
        dkt = (C.c_int32 * (3 * len(ARMS)))(*[x for a in ARMS for x in a])
        rc = C.c_int()
        self.h = self.R.ref_mab_create(dkt, len(ARMS), (C.c_int32 * len(THR))(*THR), len(THR), eps, window,
                                       C.byref(rc))
        assert rc.value == 0

    def select(self, batch, rng):
        return self.R.ref_mab_select(self.h, batch, rng)

    def record(self, s, elapsed, lens):
        b = len(lens)
        assert self.R.ref_mab_record(self.h, *s, C.c_double(elapsed), (C.c_int32 * b)(*lens), b, b) == 0


def _replay(res, prompts, max_lens, ar_tokens, seed, eps, window, threshold):
    """rollout.hpp:130-276 over the reference's select/record/step_latency."""
    R = O.ref()
    R.ref_step_latency.argtypes = [C.c_int] * 6
    root = R.ref_rng_create(seed, 0)
    sel = R.ref_rng_fork(root, 0x53454C)
    mab = _RefMab(eps, window)
    n = len(prompts)
    gen = [[] for _ in range(n)]
    running = [True] * n
    finish = [0.0] * n
    total = 0.0
    max_depth = max(a[0] for a in ARMS)
    at_least = [0] * max_depth
    trace = res["trace"]
    assert res["trace_len"] == len(trace)
    for step, m in enumerate(trace):
        active = [i for i in range(n) if running[i]]
        assert active, "GPU ran more steps than the reference loop"
        batch = len(active)
        assert m["step_index"] == step and m["batch_size"] == batch
        sd = batch < threshold  # should_enable_sd (rollout.hpp:54-57)
        assert m["sd_active"] == sd
        if sd:
            arm = mab.select(batch, sel)
            s = ARMS[arm]
            assert m["strategy"] == s, (step, m["strategy"], s)
            lens = m["accept_lens"]
            assert len(lens) == batch
            for j, i in enumerate(active):
                a = lens[j]
                assert 0 <= a <= s[0]
                for d in range(min(a, max_depth)):
                    at_least[d] += 1
                for _ in range(a + 1):  # accepted ++ bonus, cut at EOS / max_len (:231-240)
                    t = ar_tokens[i][len(gen[i])]
                    gen[i].append(t)
                    if t == 0 or len(gen[i]) >= max_lens[i]:
                        running[i] = False
                        break
            elapsed = R.ref_step_latency(batch, s[2], s[0], s[1], s[2], 1)
            mab.record(s, elapsed, lens)
        else:
            assert m["strategy"] is None
            for i in active:
                t = ar_tokens[i][len(gen[i])]
                gen[i].append(t)
                if t == 0 or len(gen[i]) >= max_lens[i]:
                    running[i] = False
            elapsed = R.ref_step_latency(batch, 1, 0, 0, 0, 0)
        assert m["elapsed"] == elapsed, (step, m["elapsed"], elapsed)
        total += elapsed
        for i in active:
            if not running[i] and finish[i] == 0.0:
                finish[i] = total
    assert not any(running)
    return gen, finish, total, at_least


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref (reference bridge) not built")
@pytest.mark.parametrize("use_graphs", [True, False])
def test_mab_rollout_replays_reference_run_rollout(omodel, use_graphs):
    rng = np.random.default_rng(3)
    n = 6
    prompts = [rng.integers(2, TINY["vocab"], 12).tolist() for _ in range(n)]
    max_lens = [14, 30, 47, 60, 75, 96]
    eps, window, seed, thr = 0.1, 20, 5, 32
    eng = Engine("tiny", max_slots=n, max_ctx=512)
    mab = Mab(ARMS, THR, eps, window)
    res = eng.run_rollout(prompts, max_lens, enable_sd=True, elastic_threshold=thr, mab=mab, seed=seed,
                          use_graphs=use_graphs, parity_elapsed=True)
    # the replay emits from the GPU's own stream (the emission / EOS / max_len
    # cut and the step loop are what is replayed); the stream itself must be
    # the oracle's greedy decode, modulo floating-point near-ties
    gen, finish, total, at_least = _replay(res, prompts, max_lens, res["tokens"], seed, eps, window, thr)
    assert res["tokens"] == gen
    from parity_util import greedy_streams_agree
    for p, ml, toks in zip(prompts, max_lens, res["tokens"]):
        ok, k, margin = greedy_streams_agree(omodel, p, toks, _oracle_ar(omodel, p, ml), TINY["vocab"])
        assert ok, (k, margin)
    assert res["finish_time"] == finish
    assert res["total_time"] == total
    assert res["accept_at_least"] == at_least
    assert res["sd_steps"] == sum(1 for m in res["trace"] if m["sd_active"])
    assert res["plain_steps"] == len(res["trace"]) - res["sd_steps"]
    assert res["verify_events"] == sum(len(m["accept_lens"]) for m in res["trace"] if m["sd_active"])
    assert res["accepted_total"] == sum(sum(m["accept_lens"]) for m in res["trace"] if m["sd_active"])
    assert res["ngram_verify_events"] == 0
    assert len({m["strategy"] for m in res["trace"] if m["sd_active"]}) >= 2  # the bandit explored
    eng.close()


def test_measured_elapsed_feeds_the_trace():
    """parity_elapsed = 0 (the product setting): elapsed = device ms."""
    rng = np.random.default_rng(4)
    prompts = [rng.integers(2, TINY["vocab"], 10).tolist() for _ in range(3)]
    eng = Engine("tiny", max_slots=3, max_ctx=256)
    res = eng.run_rollout(prompts, [20, 25, 30], enable_sd=True, elastic_threshold=2, strategy=(4, 4, 16))
    assert res["trace"][0]["sd_active"] is False  # batch 3 >= threshold 2: plain decode first
    assert any(m["sd_active"] for m in res["trace"])
    for m in res["trace"]:
        assert m["elapsed"] == m["device_ms"] and m["elapsed"] > 0
    assert abs(res["total_time"] - sum(m["elapsed"] for m in res["trace"])) < 1e-6 * res["total_time"]
    assert max(res["finish_time"]) == res["total_time"]
    eng.close()


def test_custom_cost_model_and_ngram_counters():
    """A non-default CostModelParams reaches step_latency; n-gram verify
    events are counted (rollout.hpp:226)."""
    rng = np.random.default_rng(5)
    prompts = [(rng.integers(2, 40, 6).tolist() * 4) for _ in range(2)]
    eng = Engine("tiny", max_slots=2, max_ctx=256)
    cost = CostModel(0.5, 2.0, 1.0, 1.0, 100.0, 0.25)
    res = eng.run_rollout(prompts, [24, 24], enable_sd=True, elastic_threshold=8, strategy=(4, 1, 4),
                          parity_elapsed=True, cost=cost, drafter_stale=True)
    for m in res["trace"]:
        b = m["batch_size"]
        want = 0.5 + max(2.0, b * 4 / 100.0) + 4 * 0.25
        assert m["elapsed"] == want and m["via_ngram"]
    assert res["ngram_verify_events"] == res["verify_events"] > 0
    eng.close()


def test_keep_finished_exports_truncated_sequence():
    """finished requests stay exportable (C2) after the rollout;
    the export holds exactly prompt ++ generated (cut at max_len)."""
    rng = np.random.default_rng(6)
    prompts = [rng.integers(2, TINY["vocab"], 9).tolist() for _ in range(3)]
    max_lens = [7, 19, 33]
    eng = Engine("tiny", max_slots=3, max_ctx=256)
    res = eng.run_rollout(prompts, max_lens, enable_sd=True, elastic_threshold=8, strategy=(6, 4, 24),
                          keep_finished=True)
    for i in range(3):
        toks, feats = eng.export_sequence(i)
        want = prompts[i] + res["tokens"][i]
        assert toks.tolist() == want
        assert feats.shape[0] == len(want) - 1
        eng.release(i)
    eng.close()
