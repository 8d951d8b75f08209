"""Floating-point parity of the neural leaves at the BASELINE config-2 shape
(Qwen2.5-7B-shaped target, 28 layers, V = 152064, random-init bf16 weights):
GPU logits, drafter rows and target hidden states vs the CPU neural oracle
(oracle/orc_neural.c: fp32 arithmetic over the same bf16 weights, bf16
rounding at the same points as the engine).

Stated tolerances (bf16 activations, fp32 accumulation in a different order
on each side; a near-tie of an fp32 value at a bf16 rounding boundary flips
one activation by one bf16 ulp and the flip propagates through the layers):
  logits          |gpu - cpu| <= 0.05 + 0.01 |cpu|
  drafter rows    |log p_gpu - log p_cpu| <= 0.2 where p_cpu > 1e-6
  hidden states   |gpu - cpu| <= 0.05 rms(row) + 0.02 |cpu| elementwise and
                  mean |gpu - cpu| <= 0.01 rms(row)  (bf16 features after 28
                  layers: measured max 0.19 at rms ~6, i.e. a few bf16 ulps)
The discrete decisions these feed are checked bit-exact elsewhere
(test_gpu_parity_graphs.py, oracle in the loop)."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle as O
from paper_2511_16665_b200.engine import INITS, MODELS, Engine
from parity_util import tree_paths

pytestmark = pytest.mark.gpu
M7 = MODELS["qwen2.5-7b"]
I7 = INITS["qwen2.5-7b"]
V = M7["vocab"]
P = 24
LOGIT_ATOL, LOGIT_RTOL = 0.05, 0.01


@pytest.fixture(scope="module")
def o7b():
    L = O.orc()
    cfg = O.ModelCfg(V, M7["hidden"], M7["layers"], M7["heads"], M7["kv_heads"], M7["head_dim"], M7["ffn"],
                     M7["qkv_bias"], M7["rope_theta"], M7["rms_eps"], 128)
    ini = O.InitCfg(I7["seed"], I7["layer_scale"], I7["lm_gain"], I7["lm_alt"], I7["lm_noise"], I7["fc_noise"],
                    int(I7.get("drafter_lm_fp8", 0)))
    m = L.orc_model_create(C.byref(cfg), C.byref(ini), os.cpu_count() or 8)
    assert m
    yield m
    L.orc_model_destroy(m)


def _seq(m, prompt):
    L = O.orc()
    s = L.orc_seq_create(m)
    L.orc_seq_append.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
    arr = (C.c_int32 * len(prompt))(*prompt)
    assert L.orc_seq_append(s, arr, len(prompt)) == 0
    return s


def _logits(s, path=()):
    L = O.orc()
    out = np.zeros(V, np.float32)
    p = (C.c_int32 * max(1, len(path)))(*path)
    L.orc_target_logits_path.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    assert L.orc_target_logits_path(s, p, len(path), out.ctypes.data_as(C.c_void_p)) == 0
    return out


def _drafter_row(s, path=()):
    L = O.orc()
    out = np.zeros(V, np.float64)
    p = (C.c_int32 * max(1, len(path)))(*path)
    L.orc_drafter_row.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    assert L.orc_drafter_row(s, p, len(path), out.ctypes.data_as(C.c_void_p), None) == 0
    return out


def _close(gpu, cpu, what):
    err = np.abs(gpu - cpu)
    bound = LOGIT_ATOL + LOGIT_RTOL * np.abs(cpu)
    assert np.all(err <= bound), f"{what}: max |d| {err.max():.4f} (worst excess {(err - bound).max():.4f})"
    return float(err.max())


def _bf16(bits):
    return (np.asarray(bits, np.uint32) << 16).view(np.float32)


def test_7b_logits_rows_and_hidden_states_match_oracle(o7b):
    L = O.orc()
    rng = np.random.default_rng(21)
    prompts = [rng.integers(2, V, P).tolist() for _ in range(2)]
    eng = Engine("qwen2.5-7b", max_slots=2, max_ctx=128)
    eng.set_debug(True)
    eng.prefill([0, 1], prompts)
    strategy = (4, 8, 16)
    r = eng.sd_step(strategy, [0, 1])
    errs = []
    for i, p in enumerate(prompts):
        s = _seq(o7b, p)
        vl = eng.debug_verify_logits(i)
        paths = tree_paths(r.tree[i])
        errs.append(_close(vl[0], _logits(s), f"req {i} root logits"))
        for nd in sorted({0, 1, 5, len(paths) - 1}):
            errs.append(_close(vl[1 + nd], _logits(s, paths[nd]), f"req {i} tree node {nd} logits"))
        for path, row in eng.debug_expansions(i)[:4]:
            ref = _drafter_row(s, path)
            m = ref > 1e-6
            d = np.abs(np.log(row[m]) - np.log(ref[m]))
            assert d.max() < 0.2, (i, path, float(d.max()))
        # target hidden states of the prompt positions (drafter features, C2 payload)
        toks, feats = eng.export_sequence(i, device=False)
        n = P - 1
        assert toks[:P].tolist() == p
        ref = np.zeros((n, M7["hidden"]), np.uint16)
        L.orc_seq_features.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        assert L.orc_seq_features(s, 0, n, ref.ctypes.data_as(C.c_void_p)) == 0
        g = feats[:n].view(dtype=__import__("torch").int16).numpy().view(np.uint16)
        gf, cf = _bf16(g), _bf16(ref)
        rms = np.sqrt(np.mean(cf.astype(np.float64) ** 2, axis=1, keepdims=True))
        err = np.abs(gf - cf)
        assert np.all(err <= 0.05 * rms + 0.02 * np.abs(cf)), (i, float(err.max()), float(rms.max()))
        assert np.all(err.mean(axis=1, keepdims=True) <= 0.01 * rms), (i, float(err.mean()))
        print(f"req {i} hidden states: max |dh| {err.max():.4f}, mean |dh| / rms {float((err / rms).mean()):.5f}")
        L.orc_seq_destroy(s)
    # plain decode logits (the AR denominator's LM head)
    for sl in (0, 1):
        eng.release(sl)
    eng.prefill([0, 1], prompts)
    toks, _ = eng.ar_step([0, 1])
    lg = eng.debug_ar_logits(2)
    for i, p in enumerate(prompts):
        s = _seq(o7b, p)
        ref = _logits(s)
        errs.append(_close(lg[i], ref, f"req {i} AR logits"))
        srt = np.sort(ref)
        if srt[-1] - srt[-2] > 2 * (LOGIT_ATOL + LOGIT_RTOL * abs(srt[-1])):
            assert toks[i] == int(np.argmax(ref))
        L.orc_seq_destroy(s)
    print("max |dlogit| per check:", [round(e, 4) for e in errs])
    eng.close()
