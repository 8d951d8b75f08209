"""Time several GEMM shapes in one process (env knobs are read once per process).

  python tools/time_gemms.py M:K:N:kind ...   -> one line per shape
Weights rotate over 4 copies (> L2) so every launch streams them from HBM.
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2511_16665_b200 import _lib  # noqa: E402

L = _lib.lib()
ws = torch.empty(1 << 20, device="cuda", dtype=torch.float32)
for spec in sys.argv[1:]:
    m, k, n, kind = (int(a) for a in spec.split(":"))
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
    y32 = torch.empty(m, n, device="cuda", dtype=torch.float32)
    y16 = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    ms = C.c_float()
    rc = L.tlt_dev_time_gemm(x.data_ptr(), m, k, w.data_ptr(), n, kind, y32.data_ptr(), y16.data_ptr(),
                             ws.data_ptr(), ws.numel(), 30, C.byref(ms))
    flops = 2.0 * m * n * k
    byts = n * k * 2
    print(f"M={m} K={k} N={n} kind={kind} splits={rc} us={ms.value*1e3:.1f} tflops={flops/ms.value/1e9:.0f} "
          f"wGB/s={byts/ms.value/1e6:.0f}", flush=True)
