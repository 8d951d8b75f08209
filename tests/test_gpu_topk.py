"""Row top-k kernel (drafter child selection) vs a torch fp32 reference:
ids ordered by (logit desc, id asc) — the reference child order
(spec_decode.hpp:121-125) — exact; M exact; S within fp32 tolerance."""
import ctypes as C

import pytest
import torch

from paper_2511_16665_b200 import _lib

pytestmark = pytest.mark.gpu


def run(logits, k):
    R, V = logits.shape
    part = torch.empty(((V + 127) // 128) * R * (2 + 2 * k), device="cuda")
    tok = torch.empty(R, k, dtype=torch.int32, device="cuda")
    val = torch.empty(R, k, device="cuda")
    M = torch.empty(R, device="cuda")
    S = torch.empty(R, device="cuda")
    ms = C.c_float()
    rc = _lib.lib().tlt_dev_row_topk(logits.data_ptr(), R, V, k, part.data_ptr(), tok.data_ptr(), val.data_ptr(),
                                     M.data_ptr(), S.data_ptr(), 1, C.byref(ms))
    assert rc >= 1, _lib.last_error()
    torch.cuda.synchronize()
    return tok, val, M, S


def ref_topk(logits, k):
    # stable sort of -logit keeps ascending ids among equal logits
    return torch.argsort(-logits.double(), dim=1, stable=True)[:, :k]


@pytest.mark.parametrize("R,V,k", [(3, 4096, 8), (17, 152064, 8), (64, 152064, 4), (5, 1000, 2), (300, 4096, 8)])
@pytest.mark.parametrize("pattern", ["randn", "ramp", "ties"])
def test_row_topk(R, V, k, pattern):
    g = torch.Generator(device="cuda").manual_seed(R * 31 + V + k)
    if pattern == "randn":
        x = torch.randn(R, V, device="cuda", generator=g) * 3
    elif pattern == "ramp":  # monotone in id: worst case for insertion-based scans
        x = torch.arange(V, device="cuda", dtype=torch.float32).expand(R, V) * 1e-3 + torch.arange(R, device="cuda")[:, None]
        x = x.contiguous()
    else:  # heavy exact ties: lowest id must win
        x = torch.randint(0, 5, (R, V), device="cuda", generator=g).float()
    tok, val, M, S = run(x, k)
    want = ref_topk(x, k)
    assert torch.equal(tok.long(), want), (tok[:2], want[:2])
    assert torch.equal(val, torch.gather(x, 1, want))
    assert torch.equal(M, x.max(dim=1).values)
    Sref = torch.exp(x.double() - x.max(dim=1, keepdim=True).values.double()).sum(dim=1)
    assert torch.allclose(S.double(), Sref, rtol=1e-4)


def lm_topk(x, w, k, thr=None):
    m, n = x.shape[0], w.shape[0]
    part = torch.empty(((n + 127) // 128) * m * (2 + 2 * k), device="cuda")
    tok = torch.empty(m, k, dtype=torch.int32, device="cuda")
    val = torch.empty(m, k, device="cuda")
    M = torch.empty(m, device="cuda")
    S = torch.empty(m, device="cuda")
    rc = _lib.lib().tlt_dev_lm_topk(x.data_ptr(), m, x.shape[1], w.data_ptr(), n, k, part.data_ptr(), tok.data_ptr(),
                                    val.data_ptr(), M.data_ptr(), S.data_ptr(), None if thr is None else thr.data_ptr())
    assert rc >= 1, _lib.last_error()
    return tok, val, M, S


@pytest.mark.parametrize("variant", [0, 2, 3, 8])
@pytest.mark.parametrize("m,n,k", [(8, 152064, 3584), (64, 152064, 3584), (248, 152064, 3584), (496, 20000, 512),
                                   (3, 1000, 256), (130, 4100, 512)])
@pytest.mark.parametrize("topk", [8, 4, 2, 1])
@pytest.mark.parametrize("bound", [True, False])
def test_fused_lm_head_topk(monkeypatch, variant, m, n, k, topk, bound):
    """The LM head's fused top-k epilogue (drafter children, logits never in
    HBM) against the same tcgen05 GEMM's materialised fp32 logits (whole-K
    accumulators, one split): ids by (logit desc, id asc) and values exact,
    M exact, S within fp32 tolerance. bound: with the per-row running
    k-th-value bound (tiles below it stop early), reused across two calls
    on different inputs (the merge must leave it cleared)."""
    monkeypatch.setenv("TLT_GEMM_FORCE_VARIANT", str(variant))
    g = torch.Generator(device="cuda").manual_seed(m + n + topk)
    x = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda", generator=g) / k ** 0.5).to(torch.bfloat16)
    if m >= 8:  # exact ties across vocabulary tiles: duplicate weight rows
        w[n // 2] = w[3]
        w[n - 1] = w[3]
    logits = torch.empty(m, n, device="cuda")
    ws = torch.empty(1 << 20, device="cuda")
    assert _lib.lib().tlt_dev_gemm(x.data_ptr(), m, k, w.data_ptr(), n, 0, logits.data_ptr(), None, ws.data_ptr(),
                                   ws.numel(), 1) >= 1, _lib.last_error()
    thr = torch.zeros(m, dtype=torch.int32, device="cuda") if bound else None
    if bound:  # a first call on other inputs leaves bounds that must not leak
        lm_topk(torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16) * 4, w, topk, thr)
        torch.cuda.synchronize()
        assert int(thr.abs().sum()) == 0
    tok, val, M, S = lm_topk(x, w, topk, thr)
    torch.cuda.synchronize()
    want = ref_topk(logits, topk)
    assert torch.equal(tok.long(), want), (tok[:2], want[:2])
    assert torch.equal(val, torch.gather(logits, 1, want))
    assert torch.equal(M, logits.max(dim=1).values)
    Sref = torch.exp(logits.double() - logits.max(dim=1, keepdim=True).values.double()).sum(dim=1)
    assert torch.allclose(S.double(), Sref, rtol=1e-4)
