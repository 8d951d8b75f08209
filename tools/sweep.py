"""BASELINE config 5: strategy sweep (draft depth x top-k x token budget) at
batch 1/8/32/128 vs the same engine's plain AR decode, Qwen2.5-7B shape.

Writes one JSON line per (batch, strategy): device ms per SD step, mean accept
length, emitted tokens/s and the speedup over AR at that batch. Strategies
invalid for the reference capacity rule (spec_decode.hpp:36-42) are skipped.
"""
import argparse
import itertools
import json
import os
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
os.environ.setdefault("TLT_MAX_ROWS", "8192")
from paper_2511_16665_b200.engine import ConfigError, Engine  # noqa: E402


def capacity(d, k):
    tot, lvl = 0, 1
    for _ in range(d):
        lvl *= k
        tot += lvl
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--batches", type=int, nargs="*", default=[1, 8, 32, 128])
    ap.add_argument("--depths", type=int, nargs="*", default=[2, 4, 6, 8])
    ap.add_argument("--topks", type=int, nargs="*", default=[1, 2, 4, 8])
    ap.add_argument("--budgets", type=int, nargs="*", default=[16, 32, 64, 128])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/sweep.jsonl")
    a = ap.parse_args()
    bmax = max(a.batches)
    eng = Engine(a.model, max_slots=bmax, max_ctx=1024)
    rng = np.random.default_rng(0)
    prompts = [rng.integers(2, eng.vocab, 128).tolist() for _ in range(bmax)]
    eng.prefill(list(range(bmax)), prompts)
    f = open(a.out, "w")
    for b in a.batches:
        slots = list(range(b))
        ar = [eng.ar_step(slots)[1] for _ in range(a.steps + 1)][1:]
        ar_tok_s = b / (np.median(ar) / 1e3)
        rec = dict(batch=b, strategy="AR", ms=round(float(np.median(ar)), 3), tok_s=round(float(ar_tok_s), 1))
        print(json.dumps(rec), flush=True)
        f.write(json.dumps(rec) + "\n")
        for d, k, t in itertools.product(a.depths, a.topks, a.budgets):
            if t > capacity(d, k) or b * (t + 1) > 8192:
                continue
            eng.prefill(slots, prompts[:b])  # reset the contexts for every strategy
            try:
                ms, acc = [], []
                for i in range(a.steps + 1):
                    r = eng.sd_step((d, k, t), slots, want_tree=False)
                    if i:
                        ms.append(r.elapsed_ms)
                        acc.append(float(np.mean(r.accept_len)))
            except ConfigError as e:
                print(json.dumps(dict(batch=b, strategy=[d, k, t], skipped=str(e))), flush=True)
                continue
            m = float(np.median(ms))
            tok_s = b * (np.mean(acc) + 1) / (m / 1e3)
            rec = dict(batch=b, strategy=[d, k, t], ms=round(m, 3), accept=round(float(np.mean(acc)), 3),
                       tok_s=round(float(tok_s), 1), speedup_vs_ar=round(float(tok_s / ar_tok_s), 3))
            print(json.dumps(rec), flush=True)
            f.write(json.dumps(rec) + "\n")
    f.close()
    eng.close()


if __name__ == "__main__":
    main()
