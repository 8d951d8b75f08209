"""Parity on the path bench.py runs: Qwen2.5-7B-shaped target (V = 152064),
CUDA-graph replay, the reference's default BEG-MAB arms for each batch
bucket (experiment.hpp:87-95; thresholds {1,2,8,16} group T = 64/48/32/16 by
bucket, beg_mab.hpp:95-105) at b in {1, 5, 16, 31}, and SD steps that follow
plain-decode steps (the drafter catch-up of the AR -> SD transition).

Pass A runs the sequence with production graphs and no debug. Pass B resets
the slots (same prompts, deterministic prefill) and runs the same sequence
with the debug export on: its graphs are the production sequence plus
device-to-device copy nodes (drafter logits per level, verify logits, arena),
so every replayed step is checked against the C restatement of
build_draft_tree / verify_greedy fed the GPU's own rows (oracle in the loop),
and pass B's outputs must equal pass A's bit for bit."""
import numpy as np
import pytest

from paper_2511_16665_b200.engine import Engine
from parity_util import check_tree_step, same_step

pytestmark = pytest.mark.gpu
V = 152064
P = 256

# default arms per bucket (bench.DEFAULT_ARMS grouped by tokens_to_verify)
ARMS = {1: [(10, 8, 64), (6, 8, 64)], 5: [(10, 8, 48), (6, 8, 48)], 16: [(10, 8, 16), (6, 8, 16)],
        31: [(6, 8, 16), (10, 8, 16)]}


ARMS_ALL = [[(10, 8, 64), (6, 8, 64)], [(10, 8, 48), (6, 8, 48)], [(10, 8, 32), (6, 8, 32)],
            [(10, 8, 16), (6, 8, 16)]]


def _sequence(b):
    a1, a2 = ARMS[b]
    # ("ar", n) plain steps, ("sd", arm): the first SD step after AR steps runs
    # the drafter catch-up; repeated keys replay their graph
    return [("ar", 3), ("sd", a1), ("sd", a1), ("sd", a1), ("ar", 2), ("sd", a1), ("sd", a2), ("sd", a2)]


def _checked(b):
    return list(range(b)) if b <= 5 else [0, 1, b // 2, b - 1]


@pytest.mark.parametrize("b,pooled", [(1, False), (5, False), (16, False), (31, False), (5, True), (16, True),
                                      (31, True)])
def test_7b_graph_replay_default_arms_oracle_in_the_loop(b, pooled):
    """pooled: the bucketed graph pool of plan_captures is pre-built, so every
    step replays the graph of its bucket's largest batch (5 -> 7, 16/31 -> 32;
    plain decode 5 -> 8, 16 -> 16, 31 -> 32) with the padding requests inert."""
    eng = Engine("qwen2.5-7b", max_slots=32 if pooled else b, max_ctx=P + 160)
    if pooled:
        st = eng.graph_pool_build([a for arms in ARMS_ALL for a in arms], [1, 2, 8, 16], 32)
        assert st["graphs"] > 0 and st["skipped"] == 0
    rng = np.random.default_rng(100 + b)
    prompts = [rng.integers(2, V, P).tolist() for _ in range(b)]
    slots = list(range(b))
    passes = []
    for debug in (False, True):
        for s in slots:
            eng.release(s)
        eng.set_debug(debug)
        eng.prefill(slots, prompts)
        lens = [eng.slot_len(s) for s in slots]
        outs = []
        for n_step, (kind, arg) in enumerate(_sequence(b)):
            if kind == "ar":
                for _ in range(arg):
                    toks, _ = eng.ar_step(slots)
                    outs.append(("ar", toks.tolist()))
                    lens = [x + 1 for x in lens]
                continue
            r = eng.sd_step(arg, slots)
            outs.append(("sd", r))
            if debug:
                for i in _checked(b):
                    check_tree_step(eng, arg, r, i, V, lens[i], tag=(b, n_step, arg))
            lens = [int(x) for x in r.kv_len]
        passes.append(outs)
    for (ka, ra), (kb, rb) in zip(*passes):
        assert ka == kb
        if ka == "ar":
            assert ra == rb
        else:
            same_step(ra, rb)
    if pooled:  # every step replayed a pre-built graph: nothing was captured on demand
        st = eng.graph_pool_stats()
        assert st["live_graphs"] == st["graphs"]  # production graphs (debug-export graphs not counted)
    eng.close()
