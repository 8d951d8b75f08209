"""Which arm of the run_experiment step-0 workload deviates from the CPU oracle?"""
import ctypes as C
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import oracle as O  # noqa: E402
from paper_2511_16665_b200 import experiment as X  # noqa: E402
from paper_2511_16665_b200.engine import INITS, MODELS, Engine, Mab, Rng  # noqa: E402

c = X.config_from_json({"rl_steps": 1, "workload": {"requests_per_step": 12, "max_len": 64, "mu": 3.5, "prompt_len": 8}})
root = Rng(c["seed"], 0)
len_rng, prompt_rng = root.fork(100), root.fork(200)
prompts, max_lens = [], []
for _ in range(12):
    prompts.append([2 + prompt_rng.uniform_int(4094) for _ in range(8)])
    max_lens.append(X.sample_response_length(3.5, 1.0, 64, len_rng))
print("max_lens", max_lens)
T, I = MODELS["tiny"], INITS["tiny"]
L = O.orc()
cfg = O.ModelCfg(T["vocab"], T["hidden"], T["layers"], T["heads"], T["kv_heads"], T["head_dim"], T["ffn"], T["qkv_bias"],
                 T["rope_theta"], T["rms_eps"], 1024)
ini = O.InitCfg(I["seed"], I["layer_scale"], I["lm_gain"], I["lm_alt"], I["lm_noise"], I["fc_noise"],
                    int(I.get("drafter_lm_fp8", 0)))
m = L.orc_model_create(C.byref(cfg), C.byref(ini), 8)
L.orc_neural_generate_ar.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]
orc = []
for p, ml in zip(prompts, max_lens):
    out = (C.c_int32 * 128)()
    g = L.orc_neural_generate_ar(m, (C.c_int32 * 8)(*p), 8, ml, out)
    orc.append(list(out[:g]))
strategies = [tuple(s) for s in c["strategies"]]
for mode in ["nopool", "pool", "vanilla_then_pool"]:
    eng = Engine("tiny", max_slots=32, max_ctx=232)
    if mode == "vanilla_then_pool":
        eng.graph_pool_build(strategies, [1, 2, 8, 16], 32, vanilla=True)
    if mode != "nopool":
        eng.graph_pool_build(strategies, [1, 2, 8, 16], 32)
    base = eng.run_rollout(prompts, max_lens, enable_sd=False)
    tlt = eng.run_rollout(prompts, max_lens, enable_sd=True, mab=Mab(strategies, [1, 2, 8, 16], 0.1, 20), seed=5)
    bd = [i for i in range(12) if base["tokens"][i] != orc[i]]
    td = [i for i in range(12) if tlt["tokens"][i] != orc[i]]
    print(mode, "AR != oracle:", bd, "SD != oracle:", td, flush=True)
    for i in td[:3]:
        a, o = tlt["tokens"][i], orc[i]
        k = next((j for j in range(min(len(a), len(o))) if a[j] != o[j]), None)
        print("   req", i, "pos", k, "sd", a[:k + 3] if k is not None else a, "orc", o[:k + 3] if k is not None else o)
        print("   trace", [(t["batch_size"], t["strategy"]) for t in tlt["trace"][:4]])
    eng.close()
