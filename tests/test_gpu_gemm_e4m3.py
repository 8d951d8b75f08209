"""e4m3 (FP8) tcgen05 GEMM (kind::f8f6f4) vs a torch fp32 reference of the
same op: per-row e4m3 quantisation (scale = amax / 448, round-to-nearest-even,
saturating) is checked bit-exact against torch's float8_e4m3fn cast of the
same scaled values; y = (qx qw^T) * sx * sw within 1e-3 relative."""
import pytest
import torch

from paper_2511_16665_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,k,n", [(1, 256, 4096), (17, 3584, 8192), (96, 512, 1000), (240, 3584, 20000),
                                   (496, 256, 152064), (1000, 512, 4608), (8, 3584, 152064), (64, 1024, 1000),
                                   (3, 8448, 512)])
def test_gemm_e4m3(m, k, n):
    g = torch.Generator(device="cuda").manual_seed(m + k + n)
    x = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    y = torch.full((m, n), float("nan"), device="cuda")
    qx = torch.empty(m, k, dtype=torch.uint8, device="cuda")
    qw = torch.empty(n, k, dtype=torch.uint8, device="cuda")
    sx = torch.empty(m, device="cuda")
    sw = torch.empty(n, device="cuda")
    rc = _lib.lib().tlt_dev_gemm_e4m3(x.data_ptr(), m, k, w.data_ptr(), n, y.data_ptr(), qx.data_ptr(),
                                      sx.data_ptr(), qw.data_ptr(), sw.data_ptr())
    assert rc >= 1, _lib.last_error()
    for t, q, s in ((x, qx, sx), (w, qw, sw)):
        amax = t.float().abs().amax(dim=1)
        # IEEE fp32 division (torch turns "tensor / scalar" into a reciprocal multiply)
        s_ref = torch.where(amax > 0, (amax.double() / 448.0).float(), torch.ones_like(amax))
        assert torch.equal(s, s_ref)
        q_ref = (t.double() / s_ref.double()[:, None]).float().to(torch.float8_e4m3fn).view(torch.uint8)
        assert torch.equal(q, q_ref)
    dq_x = qx.view(torch.float8_e4m3fn).float() * sx[:, None]
    dq_w = qw.view(torch.float8_e4m3fn).float() * sw[:, None]
    ref = dq_x @ dq_w.t()
    err = (y - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), err
