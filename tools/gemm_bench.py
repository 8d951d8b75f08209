"""Micro-benchmark of the tcgen05 GEMM at the Qwen2.5-7B verify shapes (CUDA events)."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2511_16665_b200 import _lib  # noqa: E402

PEAK_GBS = 6555.5
PEAK_TF = 1629.1
SHAPES = {"qkv": (3584, 4608), "o": (3584, 3584), "gate_up": (3584, 37888), "down": (18944, 3584),
          "lm_head": (3584, 152064)}


def main():
    L = _lib.lib()
    ws = torch.empty(256 << 20, device="cuda", dtype=torch.float32)
    res = []
    for m in [int(a) for a in (sys.argv[1:] or ["1", "17", "65", "256", "528"])]:
        for name, (k, n) in SHAPES.items():
            x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
            w = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
            y = torch.empty(m, n, device="cuda", dtype=torch.float32)
            args = (x.data_ptr(), m, k, w.data_ptr(), n, 0, y.data_ptr(), None, ws.data_ptr(), ws.numel(), 0)
            splits = L.tlt_dev_gemm(*args)
            assert splits >= 1, _lib.last_error()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            ev0.record()
            for _ in range(reps):
                L.tlt_dev_gemm(*args)
            ev1.record()
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1) / reps  # includes a host sync per call
            byts = n * k * 2 + m * k * 2 + m * n * 4
            flops = 2.0 * m * n * k
            res.append(dict(m=m, op=name, splits=splits, ms=round(ms, 4), gbs=round(byts / ms / 1e6, 1),
                            hbm_frac=round(byts / ms / 1e6 / PEAK_GBS, 3), tflops=round(flops / ms / 1e9, 1),
                            tc_frac=round(flops / ms / 1e9 / PEAK_TF, 3)))
            print(json.dumps(res[-1]), flush=True)


if __name__ == "__main__":
    main()
