"""The split boundary (tlt_draft / tlt_verify_accept_commit), the per-request
reference seam (DraftPlanner + verify_greedy, spec_decode.hpp:319-341 and
:245-268) and its executed reference-side adapter.

  * draft + verify(engine tree) and draft + verify(host copy of the tree)
    reproduce the fused tlt_sd_step bit for bit (same engine state);
  * an arbitrary host tree is verified with the reference's greedy rule:
    the accepted path follows the target's argmax (plain-decode tokens),
    the lowest-index child wins among equal-token siblings, the bonus is the
    argmax at the divergence, and the KV commit keeps later steps exact;
  * oracle/_ref/adapter_run (the unmodified reference types driving the
    engine through include/tlt_specsim.hpp in spec_generate's loop) emits
    exactly the CPU neural oracle's spec_generate tokens.
"""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import oracle as O
from paper_2511_16665_b200.engine import INITS, MODELS, ConfigError, Engine
from parity_util import same_step

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _prompts(b, P, V, seed):
    rng = np.random.default_rng(seed)
    return [rng.integers(2, V, P).tolist() for _ in range(b)]


@pytest.mark.parametrize("model,b,strategy", [("tiny", 4, (4, 4, 16)), ("tiny", 3, (5, 2, 12)),
                                              ("qwen2.5-7b", 3, (6, 8, 16))])
def test_split_equals_fused(model, b, strategy):
    eng = Engine(model, max_slots=b, max_ctx=256)
    V = eng.vocab
    prompts = _prompts(b, 24, V, 3)
    slots = list(range(b))
    runs = []
    for mode in ("fused", "split_device", "split_host"):
        for s in slots:
            eng.release(s)
        eng.prefill(slots, prompts)
        outs = []
        for step in range(3):
            if mode == "fused":
                r = eng.sd_step(strategy, slots)
            else:
                trees = eng.draft(strategy, slots)
                again = eng.draft(strategy, slots)  # drafting twice is idempotent
                assert again == trees
                if mode == "split_device":
                    r = eng.verify(slots, draft_depth=strategy[0])
                else:
                    r = eng.verify(slots, trees=trees)
                    # host-tree accept arrays are [b][stride]; same values
                r.tree = trees
            outs.append(r)
        runs.append(outs)
    for a, b_ in zip(runs[0], runs[1]):
        same_step(a, b_)
    for a, b_ in zip(runs[0], runs[2]):
        same_step(a, b_)
    eng.close()


def test_verify_arbitrary_host_tree():
    """Hand-built trees vs the target's greedy continuation (plain decode)."""
    eng = Engine("tiny", max_slots=2, max_ctx=256)
    V = eng.vocab
    prompts = _prompts(2, 20, V, 9)
    eng.prefill([0, 1], prompts)
    cont = [[], []]
    for _ in range(5):
        t, _ = eng.ar_step([0, 1])
        for i in range(2):
            cont[i].append(int(t[i]))
    for s in (0, 1):
        eng.release(s)
    eng.prefill([0, 1], prompts)
    # continuation c = [c0 .. c4]: the argmax at the root is c0, after c0 it is c1, ...
    wrong = [next(w for w in range(2, V) if w not in c) for c in cont]
    c = cont
    trees = [
        # request 0: wrong child, right child c0 -> c1 -> (wrong, c2 ; duplicate c2 later)
        [(wrong[0], -1), (c[0][0], -1), (c[0][1], 1), (wrong[0], 2), (c[0][2], 2), (c[0][2], 2)],
        # request 1: a chain that diverges after two tokens
        [(c[1][0], -1), (c[1][1], 0), (wrong[1], 1)],
    ]
    r = eng.verify([0, 1], trees=trees)
    assert r.accepted[0] == c[0][:3] and r.nodes[0] == [1, 2, 4]  # lowest-index child among equal tokens
    assert int(r.bonus[0]) == c[0][3]
    assert r.accepted[1] == c[1][:2] and r.nodes[1] == [0, 1]
    assert int(r.bonus[1]) == c[1][2]
    assert r.kv_len.tolist() == [20 + 3, 20 + 2]
    # the commit left exact state: the next plain step continues the greedy stream
    t, _ = eng.ar_step([0, 1])
    assert int(t[0]) == c[0][4] and int(t[1]) == c[1][3]
    # empty tree = a plain step emitting the bonus
    r = eng.verify([0, 1], trees=[[], []])
    assert r.accept_len.tolist() == [0, 0]
    # malformed trees are ConfigError (reference errors.hpp)
    with pytest.raises(ConfigError):
        eng.verify([0], trees=[[(5, 0)]])  # parent must precede the child
    with pytest.raises(ConfigError):
        eng.verify([0], trees=[[(V, -1)]])  # token out of range
    with pytest.raises(ConfigError):
        eng.verify([1], draft_depth=4)  # no tlt_draft of this slot
    eng.close()


ADAPTER = os.path.join(ROOT, "oracle", "_ref", "adapter_run")


@pytest.mark.skipif(not os.path.exists(ADAPTER), reason="adapter_run not built (needs the reference headers)")
@pytest.mark.parametrize("strategy", [(4, 4, 16), (3, 2, 6)])
def test_reference_adapter_runs_spec_generate_on_gpu(strategy):
    tiny, ini = MODELS["tiny"], INITS["tiny"]
    prompt = _prompts(1, 16, tiny["vocab"], 17)[0]
    max_len = 48
    out = subprocess.run([ADAPTER, str(max_len), *map(str, strategy), *map(str, prompt)], capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = dict(line.split(" ", 1) for line in out.stdout.strip().splitlines())
    gpu = [int(x) for x in lines["tokens"].split()]
    L = O.orc()
    cfg = O.ModelCfg(tiny["vocab"], tiny["hidden"], tiny["layers"], tiny["heads"], tiny["kv_heads"],
                     tiny["head_dim"], tiny["ffn"], tiny["qkv_bias"], tiny["rope_theta"], tiny["rms_eps"], 512)
    icfg = O.InitCfg(ini["seed"], ini["layer_scale"], ini["lm_gain"], ini["lm_alt"], ini["lm_noise"], ini["fc_noise"],
                    int(ini.get("drafter_lm_fp8", 0)))
    m = L.orc_model_create(C.byref(cfg), C.byref(icfg), 4)
    L.orc_neural_spec_generate.argtypes = [C.c_void_p] * 11
    pa = (C.c_int32 * len(prompt))(*prompt)
    o = (C.c_int32 * 256)()
    n = C.c_int()
    acc = (C.c_int32 * 256)()
    steps = L.orc_neural_spec_generate(m, pa, len(prompt), max_len, C.byref(O.Strategy(*strategy)), o, C.byref(n),
                                       acc, None, None, 256)
    assert steps > 0
    assert gpu == list(o[:n.value])
    assert [int(x) for x in lines["accept_lens"].split()] == list(acc[:steps])
    L.orc_model_destroy(m)
