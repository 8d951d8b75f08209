"""BASELINE config 4 (bounded sample): Qwen2.5-32B-shaped random-init target +
1-layer drafter, stochastic linear-chain SD (rejection sampling, seeded
RngStream uniforms), temperature 0.9, BEG-MAB over D in {4,6,8} (k=1, T=D),
long-tail rollout of 32 requests with the CUDA-graph pool, vs the same
engine's sampled plain decode on the same workload. One JSON line.

Default: the stated shape — lengths lognormal(ln 3000, 1.0) capped at 16384
— with 16 requests (the per-slot KV pool of 32 x 16.6k positions, 139 GB,
does not fit next to 65.5 GB of weights; "cap the bucket max
batch"). --bounded: 32 requests, lognormal(ln 600, 1) capped at 4096."""
import json
import math
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from bench import response_lengths  # noqa: E402
from paper_2511_16665_b200.engine import Engine, Mab  # noqa: E402

ARMS = [(8, 1, 8), (6, 1, 6), (4, 1, 4)]
bounded = "--bounded" in sys.argv
n, prompt = (32, 256) if bounded else (16, 256)
median, max_len = (600, 4096) if bounded else (3000, 16384)
eng = Engine("qwen2.5-32b", max_slots=n, max_ctx=prompt + max_len + 16)
rng = np.random.default_rng(0)
prompts = [rng.integers(2, eng.vocab, prompt).tolist() for _ in range(n)]
lens = response_lengths(n, math.log(median), 1.0, max_len, seed=4)
mab = Mab(ARMS, [1, 2, 8], 0.1, 20)
out = {}
for name, sd in ([("sd_warm", True), ("sd", True), ("ar", False)] if bounded else [("sd", True), ("ar", False)]):
    r = eng.run_rollout(prompts, lens, enable_sd=sd, elastic_threshold=32 + 1, mab=mab if sd else None,
                        strategy=(4, 1, 4), seed=1, use_graphs=True, mode="stochastic" if sd else "greedy",
                        temperature=0.9)
    out[name] = dict(tok_s=r["emitted_total"] / (r["device_ms"] / 1e3), emitted=r["emitted_total"],
                     device_ms=r["device_ms"], sd_steps=r["sd_steps"], plain_steps=r["plain_steps"],
                     mean_accept=(r["accepted_total"] / r["verify_events"]) if r["verify_events"] else None)
    print(name, json.dumps(out[name]), file=sys.stderr, flush=True)
print(json.dumps({"workload": f"config4 ({'bounded' if bounded else 'stated shape'}): qwen2.5-32b random-init, "
                              f"{n} requests, stochastic linear chains t=0.9, BEG-MAB D in {{4,6,8}}, "
                              f"lognormal(ln {median}, 1) max {max_len}, SD for every batch",
                  "lengths": {"max": max(lens), "mean": sum(lens) / len(lens)},
                  "sd_tokens_per_s": round(out["sd"]["tok_s"], 1), "ar_sampled_tokens_per_s": round(out["ar"]["tok_s"], 1),
                  "speedup": round(out["sd"]["tok_s"] / out["ar"]["tok_s"], 3),
                  "mean_accept_len": out["sd"]["mean_accept"], "sd_steps": out["sd"]["sd_steps"],
                  "ar_steps": out["ar"]["plain_steps"]}))
eng.close()
