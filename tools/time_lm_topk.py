"""Drafter LM head at k = 8: fused top-k epilogue (tlt_dev_lm_topk) vs fp32
logits + chunked row top-k (tlt_dev_gemm + tlt_dev_row_topk); wall time per
call incl. one device sync each (both paths pay it)."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2511_16665_b200 import _lib  # noqa: E402

L = _lib.lib()
V, D, K = 152064, 3584, 8
w = (torch.randn(V, D, device="cuda") / D ** 0.5).to(torch.bfloat16)
ws = torch.empty(1 << 20, device="cuda")
for m in [8, 64, 128, 248, 496]:
    x = torch.randn(m, D, device="cuda").to(torch.bfloat16)
    part = torch.empty(((V + 127) // 128) * m * (2 + 2 * K), device="cuda")
    tok = torch.empty(m, K, dtype=torch.int32, device="cuda")
    val = torch.empty(m, K, device="cuda")
    M = torch.empty(m, device="cuda")
    S = torch.empty(m, device="cuda")
    logits = torch.empty(m, V, device="cuda")
    ms = C.c_float()
    thr = torch.zeros(m, dtype=torch.int32, device="cuda")

    def fused():
        assert L.tlt_dev_lm_topk(x.data_ptr(), m, D, w.data_ptr(), V, K, part.data_ptr(), tok.data_ptr(),
                                 val.data_ptr(), M.data_ptr(), S.data_ptr(), thr.data_ptr()) >= 1

    def fused_nobound():
        assert L.tlt_dev_lm_topk(x.data_ptr(), m, D, w.data_ptr(), V, K, part.data_ptr(), tok.data_ptr(),
                                 val.data_ptr(), M.data_ptr(), S.data_ptr(), None) >= 1

    def unfused():
        assert L.tlt_dev_gemm(x.data_ptr(), m, D, w.data_ptr(), V, 0, logits.data_ptr(), None, ws.data_ptr(),
                              ws.numel(), 1) >= 1
        assert L.tlt_dev_row_topk(logits.data_ptr(), m, V, K, part.data_ptr(), tok.data_ptr(), val.data_ptr(),
                                  M.data_ptr(), S.data_ptr(), 1, C.byref(ms)) >= 1

    res = {}
    for name, f in [("fused", fused), ("fused_nobound", fused_nobound), ("unfused", unfused)]:
        for _ in range(3):
            f()
        t0 = time.perf_counter()
        for _ in range(20):
            f()
        res[name] = (time.perf_counter() - t0) / 20 * 1e6
    print(f"m={m}: fused {res['fused']:.0f} us  fused w/o bound {res['fused_nobound']:.0f} us  "
          f"unfused {res['unfused']:.0f} us", flush=True)
