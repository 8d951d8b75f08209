"""One row top-k launch on random logits (for ncu captures): R V k."""
import ctypes as C
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2511_16665_b200 import _lib  # noqa: E402

R, V, k = (int(a) for a in sys.argv[1:4])
x = torch.randn(R, V, device="cuda") if len(sys.argv) < 5 else (torch.arange(V, device="cuda", dtype=torch.float32) * 1e-3).expand(R, V).contiguous()
part = torch.empty(((V + 127) // 128) * R * (2 + 2 * k), device="cuda")
tok = torch.empty(R, k, dtype=torch.int32, device="cuda")
val = torch.empty(R, k, device="cuda")
M = torch.empty(R, device="cuda")
S = torch.empty(R, device="cuda")
ms = C.c_float()
_lib.lib().tlt_dev_row_topk(x.data_ptr(), R, V, k, part.data_ptr(), tok.data_ptr(), val.data_ptr(), M.data_ptr(),
                            S.data_ptr(), 2, C.byref(ms))
torch.cuda.synchronize()
