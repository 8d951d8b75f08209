"""Tree-masked attention kernels (mma.sync and tcgen05/TMEM) vs a torch fp32
reference of the same op: committed prefix visible to every row, tail
entries (tree nodes) visible through each row's bitmask, GQA heads.
Tolerance: bf16 output rounding (|err| <= 2e-2 + 2e-2 |ref|)."""
import pytest
import torch

from paper_2511_16665_b200 import _lib

pytestmark = pytest.mark.gpu


def make_case(n_groups, rpr, lc, H=28, KV=4, hd=128, cap=2400, seed=0, remap_tail=False):
    """lc: committed keys, one int for every group or a per-group list (ragged)."""
    lcs = list(lc) if isinstance(lc, (list, tuple)) else [lc] * n_groups
    g = torch.Generator(device="cuda").manual_seed(seed)
    dev = "cuda"
    slots = n_groups
    kc = (torch.randn(slots, KV, cap, hd, device=dev, generator=g)).to(torch.bfloat16)
    vc = (torch.randn(slots, KV, cap, hd, device=dev, generator=g)).to(torch.bfloat16)
    R = n_groups * rpr
    q = (torch.randn(R, H * hd, device=dev, generator=g)).to(torch.bfloat16)
    # tree: row j's parent = (j - 1) // 2 (binary tree in rank order); row 0 = root
    par = [-1] + [(j - 1) // 2 for j in range(1, rpr)]
    vis = torch.zeros(rpr, rpr, dtype=torch.bool)
    for j in range(rpr):
        a = j
        while a >= 0:
            vis[j, a] = True
            a = par[a]
    mask = torch.zeros(R, 32, dtype=torch.int64)
    for j in range(rpr):
        for t in range(rpr):
            if vis[j, t]:
                mask[torch.arange(n_groups) * rpr + j, t >> 5] |= 1 << (t & 31)
    mask_dev = torch.tensor((mask & 0xFFFFFFFF).numpy().astype("uint32").view("int32"), device=dev)
    row_slot = torch.arange(n_groups, device=dev, dtype=torch.int32).repeat_interleave(rpr)
    g_slot = torch.arange(n_groups, device=dev, dtype=torch.int32)
    g_lc = torch.tensor(lcs, device=dev, dtype=torch.int32)
    tail0 = [x + 64 if remap_tail else x for x in lcs]
    g_tail0 = torch.tensor(tail0, device=dev, dtype=torch.int32)
    g_ntail = torch.full((n_groups,), rpr, device=dev, dtype=torch.int32)
    return dict(kc=kc, vc=vc, q=q, vis=vis, mask=mask_dev, row_slot=row_slot, g_slot=g_slot, g_lc=g_lc,
                g_tail0=g_tail0, g_ntail=g_ntail, n_groups=n_groups, rpr=rpr, lc=lcs, H=H, KV=KV, hd=hd, cap=cap,
                tail0=tail0)


def reference(c):
    H, KV, hd, rpr, G = c["H"], c["KV"], c["hd"], c["rpr"], c["H"] // c["KV"]
    out = torch.zeros(c["n_groups"] * rpr, H * hd, device="cuda")
    for i in range(c["n_groups"]):
        lc = c["lc"][i]
        keys = torch.cat([torch.arange(lc), c["tail0"][i] + torch.arange(rpr)]).cuda()
        for h in range(H):
            kvh = h // G
            K = c["kc"][i, kvh, keys].float()
            Vv = c["vc"][i, kvh, keys].float()
            Q = c["q"][i * rpr:(i + 1) * rpr, h * hd:(h + 1) * hd].float()
            s = Q @ K.t() / hd ** 0.5
            allowed = torch.cat([torch.ones(rpr, lc, dtype=torch.bool), c["vis"]], dim=1).cuda()
            s = s.masked_fill(~allowed, float("-inf"))
            out[i * rpr:(i + 1) * rpr, h * hd:(h + 1) * hd] = torch.softmax(s, dim=1) @ Vv
    return out


def run(c, kernel):
    out = torch.zeros(c["n_groups"] * c["rpr"], c["H"] * c["hd"], device="cuda", dtype=torch.bfloat16)
    rc = _lib.lib().tlt_dev_attention(
        c["q"].data_ptr(), c["kc"].data_ptr(), c["vc"].data_ptr(), out.data_ptr(), c["n_groups"], c["rpr"], c["H"],
        c["KV"], c["hd"], c["cap"], c["row_slot"].data_ptr(), c["mask"].data_ptr(), c["g_slot"].data_ptr(),
        c["g_lc"].data_ptr(), c["g_tail0"].data_ptr(), c["g_ntail"].data_ptr(), c["cap"], kernel)
    assert rc == 0, _lib.last_error()
    return out.float()


@pytest.mark.parametrize("n_groups,rpr,lc,remap", [(2, 17, 300, False), (3, 49, 700, False), (1, 65, 1000, True),
                                                   (2, 33, 0, False), (1, 17, 511, True)])
@pytest.mark.parametrize("kernel", [0, 1])
def test_tree_attention(n_groups, rpr, lc, remap, kernel):
    c = make_case(n_groups, rpr, lc, seed=n_groups * 100 + rpr + lc, remap_tail=remap)
    ref = reference(c)
    got = run(c, kernel)
    err = (got - ref).abs()
    assert torch.all(err <= 2e-2 + 2e-2 * ref.abs()), float(err.max())


@pytest.mark.parametrize("n_groups,lc", [(1, 1000), (5, 700), (33, 1500), (40, 300)])
def test_decode_attention_fused_combine(n_groups, lc):
    """Flash-decode kernel (1 row x 7 q-heads per request, balanced key splits)
    with the separate combine launch (kernel 2) and with the combine fused into
    the last CTA (kernel 3): both within bf16 tolerance of torch fp32, and
    bit-identical to each other (same merge arithmetic, fixed split order)."""
    c = make_case(n_groups, 1, lc, seed=7 * n_groups + lc)
    ref = reference(c)
    sep = run(c, 2)
    fused = run(c, 3)
    err = (sep - ref).abs()
    assert torch.all(err <= 2e-2 + 2e-2 * ref.abs()), float(err.max())
    assert torch.equal(sep, fused)


RAGGED = [1, 255, 257, 700, 2000, 64, 0, 1500]


@pytest.mark.parametrize("dyn", ["0", "1"])
@pytest.mark.parametrize("n_groups", [5, 8, 40])
def test_decode_attention_ragged_requests(monkeypatch, n_groups, dyn):
    """requests of one batch with different key counts get their
    own split count (per-request sizing, DYN=1) or the fixed chunk (DYN=0);
    the separate and the fused combine agree bit for bit and with torch."""
    monkeypatch.setenv("TLT_ATTN_DEC_DYN", dyn)
    lcs = [RAGGED[i % len(RAGGED)] for i in range(n_groups)]
    c = make_case(n_groups, 1, lcs, seed=31 * n_groups)
    ref = reference(c)
    sep = run(c, 2)
    fused = run(c, 3)
    err = (sep - ref).abs()
    assert torch.all(err <= 2e-2 + 2e-2 * ref.abs()), float(err.max())
    assert torch.equal(sep, fused)


@pytest.mark.parametrize("ctas,min_chunk", [("148", "256"), ("592", "64"), ("1", "256")])
@pytest.mark.parametrize("n_groups,rpr,remap", [(1, 65, True), (5, 49, False), (3, 17, True), (31, 17, False)])
def test_tree_attention_engine_split_plan(monkeypatch, n_groups, rpr, remap, ctas, min_chunk):
    """The tree kernel as the engine plans it (kernel 4): per-request split
    sizes from each request's own key count (ragged batches), requests that
    fit one split written directly by the attention kernel, the rest merged
    by the combine; every split plan within bf16 tolerance of torch."""
    monkeypatch.setenv("TLT_ATTN_TREE_CTAS", ctas)
    monkeypatch.setenv("TLT_ATTN_TREE_MIN_CHUNK", min_chunk)
    lcs = [RAGGED[(i * 3) % len(RAGGED)] for i in range(n_groups)]
    c = make_case(n_groups, rpr, lcs, seed=n_groups * 7 + rpr, remap_tail=remap)
    ref = reference(c)
    got = run(c, 4)
    err = (got - ref).abs()
    assert torch.all(err <= 2e-2 + 2e-2 * ref.abs()), float(err.max())


@pytest.mark.parametrize("n_groups,rpr,remap", [(1, 65, True), (5, 49, False), (3, 17, True), (31, 17, False),
                                                (2, 33, False)])
@pytest.mark.parametrize("ctas,min_chunk", [("296", "128"), ("1", "256"), ("592", "64")])
def test_tma_tree_attention(monkeypatch, n_groups, rpr, remap, ctas, min_chunk):
    """TMA-fed kernel (attn_tma.cu, kernel 5): 128B-swizzled 64 x 64 K/V boxes
    in an mbarrier ring, prefix and tree-tail tiles, ragged requests, every
    split plan within bf16 tolerance of torch fp32."""
    monkeypatch.setenv("TLT_ATTN_TREE_CTAS", ctas)
    monkeypatch.setenv("TLT_ATTN_TREE_MIN_CHUNK", min_chunk)
    lcs = [RAGGED[(i * 5) % len(RAGGED)] for i in range(n_groups)]
    c = make_case(n_groups, rpr, lcs, seed=n_groups * 11 + rpr, remap_tail=remap)
    ref = reference(c)
    got = run(c, 5)
    err = (got - ref).abs()
    assert torch.all(err <= 2e-2 + 2e-2 * ref.abs()), float(err.max())


@pytest.mark.parametrize("n_groups", [1, 5, 8, 40, 64])
def test_tma_decode_attention(n_groups):
    """TMA flash-decode (1 row x 7 q-heads per request): separate combine
    (kernel 5) and fused combine (kernel 6) equal each other bit for bit and
    torch within bf16 tolerance, on ragged key counts."""
    lcs = [RAGGED[(i * 3 + 1) % len(RAGGED)] for i in range(n_groups)]
    c = make_case(n_groups, 1, lcs, seed=13 * n_groups)
    ref = reference(c)
    sep = run(c, 5)
    fused = run(c, 6)
    err = (sep - ref).abs()
    assert torch.all(err <= 2e-2 + 2e-2 * ref.abs()), float(err.max())
    assert torch.equal(sep, fused)


def test_tma_tiny_head_dim():
    """hd = 64 (the tiny config): one 64-dim box per tile."""
    c = make_case(3, 17, [100, 5, 300], H=4, KV=2, hd=64, cap=512, seed=5)
    ref = reference(c)
    got = run(c, 5)
    err = (got - ref).abs()
    assert torch.all(err <= 2e-2 + 2e-2 * ref.abs()), float(err.max())


@pytest.mark.parametrize("n_groups", [1, 4, 12, 32])
def test_tma_tiny_decode(n_groups):
    """hd = 64 flash-decode (tiny config: 4 q-heads / 2 KV heads), TMA kernel
    (separate and fused combine) vs the mma.sync kernel vs torch."""
    lcs = [RAGGED[(i * 7 + 2) % len(RAGGED)] % 400 for i in range(n_groups)]
    c = make_case(n_groups, 1, lcs, H=4, KV=2, hd=64, cap=512, seed=17 * n_groups)
    ref = reference(c)
    got = run(c, 5)
    old = run(c, 2)
    err = (got - ref).abs()
    assert torch.all(err <= 2e-2 + 2e-2 * ref.abs()), float(err.max())
    err = (old - ref).abs()
    assert torch.all(err <= 2e-2 + 2e-2 * ref.abs()), float(err.max())


def _poison(c):
    """Every cache row outside a group's visible keys (committed prefix and
    tree tail) := NaN: kernels must never let an unused row reach the output
    (a masked probability of 0 times a NaN value is NaN)."""
    for i in range(c["n_groups"]):
        keep = torch.zeros(c["cap"], dtype=torch.bool)
        keep[:c["lc"][i]] = True
        keep[c["tail0"][i]:c["tail0"][i] + c["rpr"]] = True
        c["kc"][i][:, ~keep] = float("nan")
        c["vc"][i][:, ~keep] = float("nan")
    return c


@pytest.mark.parametrize("kernel", [5, 0, 4])
@pytest.mark.parametrize("n_groups,rpr,hd,H,KV", [(3, 17, 128, 28, 4), (2, 49, 128, 28, 4), (5, 1, 128, 28, 4),
                                                  (3, 17, 64, 4, 2), (4, 1, 64, 4, 2)])
def test_attention_ignores_nan_in_unused_cache_rows(kernel, n_groups, rpr, hd, H, KV):
    if kernel == 4 and rpr * H // KV <= 16:
        pytest.skip("tree-kernel entry needs > 16 query vectors")
    lcs = [(37 * (i + 1)) % 300 + 1 for i in range(n_groups)]
    c = _poison(make_case(n_groups, rpr, lcs, H=H, KV=KV, hd=hd, cap=512, seed=n_groups + rpr + hd,
                          remap_tail=True))
    ref = reference(c)
    got = run(c, kernel)
    assert torch.isfinite(got).all()
    err = (got - ref).abs()
    assert torch.all(err <= 2e-2 + 2e-2 * ref.abs()), float(err.max())


@pytest.mark.parametrize("n_groups,rpr,remap", [(1, 65, True), (5, 49, False), (3, 17, True), (31, 17, False),
                                                (2, 33, False), (4, 100, True)])
@pytest.mark.parametrize("ctas,min_chunk", [("296", "128"), ("1", "256"), ("1184", "64")])
def test_tcgen05_tree_attention(monkeypatch, n_groups, rpr, remap, ctas, min_chunk):
    """tcgen05 / TMEM tree attention (attn_tc5.cu, kernel 7): TMA ring, S and O
    in TMEM, lazy-rescaled online softmax, ragged requests and every split plan,
    within bf16 tolerance of torch fp32."""
    monkeypatch.setenv("TLT_ATTN_TREE_TC", "1")  # force it for shapes the engine routes elsewhere
    monkeypatch.setenv("TLT_ATTN_TREE_CTAS", ctas)
    monkeypatch.setenv("TLT_ATTN_TREE_MIN_CHUNK", min_chunk)
    lcs = [RAGGED[(i * 5 + 3) % len(RAGGED)] for i in range(n_groups)]
    c = make_case(n_groups, rpr, lcs, seed=n_groups * 13 + rpr, remap_tail=remap)
    ref = reference(c)
    got = run(c, 7)
    err = (got - ref).abs()
    assert torch.all(err <= 2e-2 + 2e-2 * ref.abs()), float(err.max())


@pytest.mark.parametrize("n_groups,rpr", [(3, 17), (2, 49)])
def test_tcgen05_tree_attention_nan_poisoned_cache(monkeypatch, n_groups, rpr):
    monkeypatch.setenv("TLT_ATTN_TREE_TC", "1")
    lcs = [(37 * (i + 1)) % 300 + 1 for i in range(n_groups)]
    c = _poison(make_case(n_groups, rpr, lcs, cap=512, seed=n_groups + rpr, remap_tail=True))
    ref = reference(c)
    got = run(c, 7)
    assert torch.isfinite(got).all()
    err = (got - ref).abs()
    assert torch.all(err <= 2e-2 + 2e-2 * ref.abs()), float(err.max())


def test_tcgen05_tree_attention_large_score_growth(monkeypatch):
    """Scores that grow by >> 2^8 along the keys force O rescales in TMEM."""
    monkeypatch.setenv("TLT_ATTN_TREE_TC", "1")
    c = make_case(2, 17, [900, 400], seed=3)
    ramp = torch.linspace(0.0, 6.0, c["cap"], device="cuda").view(1, 1, -1, 1)
    c["kc"] = (c["kc"].float() * (1.0 + ramp)).to(torch.bfloat16)
    ref = reference(c)
    got = run(c, 7)
    err = (got - ref).abs()
    assert torch.all(err <= 3e-2 + 3e-2 * ref.abs()), float(err.max())
