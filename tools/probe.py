"""Quick GPU probe: step latencies and acceptance of the engine at a model shape."""
import argparse
import json
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2511_16665_b200.engine import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--slots", type=int, default=64)
    ap.add_argument("--ctx", type=int, default=2048)
    ap.add_argument("--prompt", type=int, default=256)
    ap.add_argument("--layer-scale", type=float, nargs="*", default=[0.3])
    ap.add_argument("--gain", type=float, default=13.0)
    ap.add_argument("--alt", type=float, default=0.9)
    ap.add_argument("--batches", type=int, nargs="*", default=[1, 8, 16, 31, 64])
    ap.add_argument("--strategies", default="10,8,64;6,8,16;4,4,16;10,8,16")
    ap.add_argument("--steps", type=int, default=6)
    a = ap.parse_args()
    strategies = [tuple(int(x) for x in s.split(",")) for s in a.strategies.split(";")]
    for ls in a.layer_scale:
        t0 = time.time()
        eng = Engine(a.model, max_slots=a.slots, max_ctx=a.ctx, init=dict(layer_scale=ls, lm_gain=a.gain, lm_alt=a.alt))
        print(json.dumps(dict(event="create", layer_scale=ls, s=round(time.time() - t0, 2))), flush=True)
        rng = np.random.default_rng(0)
        V = eng.vocab
        prompts = [rng.integers(2, V, a.prompt).tolist() for _ in range(a.slots)]
        t0 = time.time()
        eng.prefill(list(range(a.slots)), prompts)
        print(json.dumps(dict(event="prefill", n=a.slots, s=round(time.time() - t0, 3))), flush=True)
        for b in a.batches:
            if b > a.slots:
                continue
            slots = list(range(b))
            ms = [eng.ar_step(slots)[1] for _ in range(a.steps)]
            print(json.dumps(dict(event="ar", b=b, ms=round(float(np.median(ms[1:])), 3),
                                  tok_s=round(b / np.median(ms[1:]) * 1e3, 1))), flush=True)
            if b >= 32:
                continue
            for s in strategies:
                accs, mss = [], []
                for _ in range(a.steps):
                    r = eng.sd_step(s, slots, want_tree=False)
                    accs.append(float(np.mean(r.accept_len)))
                    mss.append(r.elapsed_ms)
                med = float(np.median(mss[1:]))
                emitted = b * (np.mean(accs) + 1)
                print(json.dumps(dict(event="sd", b=b, strategy=s, ms=round(med, 3), accept=round(float(np.mean(accs)), 2),
                                      tok_s=round(emitted / med * 1e3, 1))), flush=True)
        eng.close()


if __name__ == "__main__":
    main()
