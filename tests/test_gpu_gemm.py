"""tcgen05 swap-AB GEMM vs a torch fp32 reference of the same op."""
import pytest
import torch

from paper_2511_16665_b200 import _lib

pytestmark = pytest.mark.gpu

SHAPES = [
    # (M tokens, K, N out)
    (17, 256, 512), (68, 256, 256), (4, 256, 1376), (64, 688, 256), (16, 256, 4096),
    (65, 3584, 4608), (200, 512, 640), (256, 1024, 384), (300, 512, 256), (528, 3584, 512),
    (1, 3584, 3584), (1088, 256, 256),
    # CTA-pair (cta_group::2) path: M >= 192, ragged N / M tiles
    (192, 256, 256), (193, 512, 384), (2048, 3584, 1000), (700, 1024, 4608), (4096, 256, 512),
    # CTA pair + split-K across a (2, 1, splits) cluster (few weight tiles)
    (300, 4096, 512), (527, 3584, 3584), (272, 18944, 3584), (200, 2048, 1000),
    # CTA pair with two 256-row sub-tiles per cluster (M >= 384, many weight tiles), ragged N
    (400, 512, 38000), (1000, 256, 40000),
]


@pytest.mark.parametrize("m,k,n", SHAPES)
@pytest.mark.parametrize("max_splits", [1, 0])
def test_gemm_f32(m, k, n, max_splits):
    torch.manual_seed(m * 7 + k + n)
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda") / k ** 0.5).to(torch.bfloat16)
    y = torch.full((m, n), float("nan"), device="cuda", dtype=torch.float32)
    ws = torch.empty(64 << 20, device="cuda", dtype=torch.float32)
    L = _lib.lib()
    rc = L.tlt_dev_gemm(x.data_ptr(), m, k, w.data_ptr(), n, 0, y.data_ptr(), None,
                        ws.data_ptr(), ws.numel(), max_splits)
    assert rc >= 1, _lib.last_error()
    ref = x.float() @ w.float().t()
    err = (y - ref).abs().max().item()
    assert err < 2e-3 * max(1.0, ref.abs().max().item()), (err, rc)


@pytest.mark.parametrize("m", [33, 517])
def test_gemm_swiglu(m):
    k, f = 512, 320
    torch.manual_seed(0)
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    w = (torch.randn(2 * f, k, device="cuda") / k ** 0.5).to(torch.bfloat16)
    y = torch.zeros(m, f, device="cuda", dtype=torch.bfloat16)
    ws = torch.empty(16 << 20, device="cuda", dtype=torch.float32)
    rc = _lib.lib().tlt_dev_gemm(x.data_ptr(), m, k, w.data_ptr(), 2 * f, 3, None, y.data_ptr(),
                                 ws.data_ptr(), ws.numel(), 0)
    assert rc >= 1, _lib.last_error()
    acc = x.float() @ w.float().t()
    g, u = acc[:, 0::2], acc[:, 1::2]
    ref = torch.nn.functional.silu(g) * u
    assert (y.float() - ref).abs().max().item() < 2e-2 * max(1.0, ref.abs().max().item())


@pytest.mark.parametrize("variant", [1, 2, 3, 4, 6, 7, 8])
@pytest.mark.parametrize("m,k,n", [(272, 3584, 4608), (528, 3584, 3584), (512, 1024, 2304), (1024, 512, 1536),
                                   (768, 256, 5000), (196, 18944, 512), (300, 4096, 512)])
def test_gemm_plan_variants(monkeypatch, variant, m, k, n):
    """Every plan variant the engine's autotuner can pick (deep-ring pairs,
    persistent pairs, single-CTA tiles, <=128-token pair tiles, pair split-K
    x4, weight multicast across a (2 mc, 1, 1) cluster) computes the same GEMM."""
    monkeypatch.setenv("TLT_GEMM_FORCE_VARIANT", str(variant))
    torch.manual_seed(m + k + n + variant)
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda") / k ** 0.5).to(torch.bfloat16)
    y = torch.full((m, n), float("nan"), device="cuda", dtype=torch.float32)
    ws = torch.empty(64 << 20, device="cuda", dtype=torch.float32)
    rc = _lib.lib().tlt_dev_gemm(x.data_ptr(), m, k, w.data_ptr(), n, 0, y.data_ptr(), None, ws.data_ptr(),
                                 ws.numel(), 0)
    assert rc >= 1, _lib.last_error()
    ref = x.float() @ w.float().t()
    err = (y - ref).abs().max().item()
    assert err < 2e-3 * max(1.0, ref.abs().max().item()), (err, rc)


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4, 6, 7, 8])
@pytest.mark.parametrize("m,k,n,live", [(1024, 512, 1536, 130), (1024, 512, 1536, 1), (528, 3584, 3584, 300),
                                        (768, 256, 5000, 767), (272, 3584, 4608, 0)])
def test_gemm_live_rows_skip(monkeypatch, variant, m, k, n, live):
    """The graph pool's padding skip (device live-row count): rows below the
    live count are exact for every plan variant, including weight multicast,
    whose (2 mc, 1, 1) cluster spans several token tiles and must skip as a
    whole (a partially live multicast cluster once wedged / faulted)."""
    monkeypatch.setenv("TLT_GEMM_FORCE_VARIANT", str(variant))
    torch.manual_seed(m + n + live + variant)
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda") / k ** 0.5).to(torch.bfloat16)
    y = torch.full((m, n), float("nan"), device="cuda", dtype=torch.float32)
    ws = torch.empty(64 << 20, device="cuda", dtype=torch.float32)
    lv = torch.tensor([live], device="cuda", dtype=torch.int32)
    for _ in range(3):
        rc = _lib.lib().tlt_dev_gemm_live(x.data_ptr(), m, k, w.data_ptr(), n, 0, y.data_ptr(), None,
                                          ws.data_ptr(), ws.numel(), lv.data_ptr())
        assert rc >= 1, _lib.last_error()
    if live:
        ref = x[:live].float() @ w.float().t()
        err = (y[:live] - ref).abs().max().item()
        assert err < 2e-3 * max(1.0, ref.abs().max().item()), (err, rc)
