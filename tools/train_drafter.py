"""Spot-train the EAGLE drafter of the 7B-shaped engine on the target's own
greedy rollouts and measure the acceptance before / after on held-out
prompts (the TLT adaptive-drafter loop on one GPU).

  python tools/train_drafter.py --iters 200 > gpurun_out/train_drafter.json
"""
import argparse
import json
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2511_16665_b200 import spot as S  # noqa: E402
from paper_2511_16665_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="qwen2.5-7b")
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--requests", type=int, default=64)
ap.add_argument("--gen", type=int, default=512)
ap.add_argument("--prompt", type=int, default=256)
ap.add_argument("--lr", type=float, default=3e-4)
ap.add_argument("--budget", type=int, default=8192)
ap.add_argument("--capacity", type=int, default=2048)
ap.add_argument("--wd", type=float, default=0.0)
a = ap.parse_args()

eng = Engine(a.model, max_slots=a.requests, max_ctx=a.prompt + a.gen + 200)
V = eng.vocab


def accept(seed, b=8, steps=8, strategy=(6, 8, 16)):
    rng = np.random.default_rng(seed)
    prompts = [rng.integers(2, V, a.prompt).tolist() for _ in range(b)]
    r = eng.run_rollout(prompts, [steps * 8] * b, enable_sd=True, elastic_threshold=1 << 20, strategy=strategy)
    return r["accepted_total"] / r["verify_events"], r["emitted_total"] / (r["device_ms"] / 1e3)


out = {"before": {str(s): accept(1000 + i, strategy=s) for i, s in enumerate([(6, 8, 16), (10, 8, 64)])}}
buf = S.DataBuffer(retention=1)
held = S.DataBuffer(retention=1)
t0 = time.time()
for step in range(3):
    rng = np.random.default_rng(step)
    prompts = [rng.integers(2, V, a.prompt).tolist() for _ in range(a.requests)]
    eng.run_rollout(prompts, [a.gen] * a.requests, enable_sd=False, keep_finished=True)
    toks, feats = [], []
    for i in range(a.requests):
        t, f = eng.export_sequence(i)
        toks.append(t.tolist())
        feats.append(f)
        eng.release(i)
    (held if step == 2 else buf).insert(min(step, 1), toks, feats)
out["collect_s"] = time.time() - t0
tr = S.DrafterTrainer(eng, lr=a.lr, weight_decay=a.wd)


def held_loss():
    import torch
    import torch.nn.functional as F
    ents = held.sample(1, 1 << 30)
    packed = S.pack_sequences([e.length() for e in ents], a.capacity)
    tot, n = 0.0, 0
    with torch.no_grad():
        for pack in packed.packs:
            tok, fp, pos, sid, lab = tr.batch_from_pack(ents, pack)
            lg = tr.forward(tok, fp, pos, sid)
            tot += float(F.cross_entropy(lg, lab, ignore_index=-100, reduction="sum"))
            n += int((lab >= 0).sum())
    return tot / n


out["held_loss_before"] = held_loss()
cfg = S.SpotTrainConfig(current_step=1, token_budget=a.budget, pack_capacity=a.capacity)
t0 = time.time()
log = S.spot_train_loop(tr, buf, cfg, a.iters)
out["train_s"] = time.time() - t0
out["loss_first"] = log.losses[:5]
out["loss_last"] = log.losses[-5:]
out["held_loss_after"] = held_loss()
out["after"] = {str(s): accept(1000 + i, strategy=s) for i, s in enumerate([(6, 8, 16), (10, 8, 64)])}
print(json.dumps(out))
eng.close()
