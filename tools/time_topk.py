"""Time the row top-k kernel on random / ramp / tie logits (data dependence check)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2511_16665_b200 import _lib  # noqa: E402

L = _lib.lib()
for R in [16, 248, 496]:
    V, k = 152064, 8
    for pat in ["randn", "ramp", "ties"]:
        if pat == "randn":
            x = torch.randn(R, V, device="cuda")
        elif pat == "ramp":
            x = (torch.arange(V, device="cuda", dtype=torch.float32) * 1e-3).expand(R, V).contiguous()
        else:
            x = torch.randint(0, 5, (R, V), device="cuda").float()
        part = torch.empty(((V + 127) // 128) * R * (2 + 2 * k), device="cuda")
        tok = torch.empty(R, k, dtype=torch.int32, device="cuda")
        val = torch.empty(R, k, device="cuda")
        M = torch.empty(R, device="cuda")
        S = torch.empty(R, device="cuda")
        ms = C.c_float()
        nch = L.tlt_dev_row_topk(x.data_ptr(), R, V, k, part.data_ptr(), tok.data_ptr(), val.data_ptr(),
                                 M.data_ptr(), S.data_ptr(), 20, C.byref(ms))
        gbs = R * V * 4 / (ms.value * 1e-3) / 1e9
        print(f"R={R} {pat:5s} nch={nch} us={ms.value * 1e3:.1f} GB/s={gbs:.0f}", flush=True)
