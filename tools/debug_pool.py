"""Repro: padded SD step (pool) vs exact step at a given batch / strategy."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2511_16665_b200.engine import Engine  # noqa: E402

ARMS = [(10, 8, 64), (6, 8, 64), (10, 8, 48), (6, 8, 48), (10, 8, 32), (6, 8, 32), (10, 8, 16), (6, 8, 16)]
b = int(sys.argv[1])
strategy = tuple(int(x) for x in sys.argv[2].split(","))
pooled = int(sys.argv[3])
graphs = int(sys.argv[4]) if len(sys.argv) > 4 else 1
rng = np.random.default_rng(b)
prompts = [rng.integers(2, 4096, 14).tolist() for _ in range(b)]
eng = Engine("tiny", max_slots=32, max_ctx=512)
if pooled:
    print(eng.graph_pool_build(ARMS, [1, 2, 8, 16], 32), flush=True)
eng.prefill(list(range(b)), prompts)
for step in range(3):
    if graphs:
        r = eng.sd_step(strategy, list(range(b)))
    else:
        eng.set_debug(True)
        r = eng.sd_step(strategy, list(range(b)))
    print("sd", r.accept_len.tolist(), flush=True)
    t, _ = eng.ar_step(list(range(b)))
    print("ar", t.tolist(), flush=True)
eng.close()
