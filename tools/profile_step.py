"""Run a bounded number of engine steps (for ncu launch lists / full captures).

  python tools/profile_step.py --model qwen2.5-7b --b 1 --ar 2 --sd 1 --strategy 6,8,16
"""
import argparse
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2511_16665_b200.engine import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--b", type=int, default=1)
    ap.add_argument("--ar", type=int, default=2)
    ap.add_argument("--sd", type=int, default=1)
    ap.add_argument("--strategy", default="6,8,16")
    ap.add_argument("--ctx", type=int, default=1024)
    ap.add_argument("--prompt", type=int, default=256)
    ap.add_argument("--graphs", type=int, default=0)
    a = ap.parse_args()
    s = tuple(int(x) for x in a.strategy.split(","))
    eng = Engine(a.model, max_slots=max(a.b, 1), max_ctx=a.ctx)
    rng = np.random.default_rng(0)
    prompts = [rng.integers(2, eng.vocab, a.prompt).tolist() for _ in range(a.b)]
    eng.prefill(list(range(a.b)), prompts)
    slots = list(range(a.b))
    for _ in range(a.ar):
        _, ms = eng.ar_step(slots)
        print("ar ms", round(ms, 3), flush=True)
    for _ in range(a.sd):
        r = eng.sd_step(s, slots, want_tree=False)
        print("sd ms", round(r.elapsed_ms, 3), "accept", r.accept_len.tolist(), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
