"""cuBLAS (torch.matmul) vs our tcgen05 GEMM on the verify / drafter shapes."""
import ctypes as C
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2511_16665_b200 import _lib  # noqa: E402

L = _lib.lib()
ws = torch.empty(1 << 22, device="cuda", dtype=torch.float32)
for spec in sys.argv[1:]:
    m, k, n = (int(a) for a in spec.split(":"))
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    ws4 = [(torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(3)]
    y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        torch.matmul(x, ws4[0].t(), out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for i in range(30):
        torch.matmul(x, ws4[i % 3].t(), out=y)
    e1.record()
    torch.cuda.synchronize()
    cub = e0.elapsed_time(e1) / 30
    y32 = torch.empty(m, n, device="cuda", dtype=torch.float32)
    ms = C.c_float()
    L.tlt_dev_time_gemm(x.data_ptr(), m, k, ws4[0].data_ptr(), n, 1, y32.data_ptr(), y.data_ptr(), ws.data_ptr(),
                        ws.numel(), 30, C.byref(ms))
    fl = 2.0 * m * n * k
    print(f"M={m} K={k} N={n}: cublas {cub*1e3:.1f} us ({fl/cub/1e9:.0f} TF/s)  ours {ms.value*1e3:.1f} us ({fl/ms.value/1e9:.0f} TF/s)", flush=True)
