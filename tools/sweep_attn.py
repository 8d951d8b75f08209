"""Attention split-plan sweep over the engine's own attention probe
(tlt_probe_attention, grid sized for the cache capacity as in the engine).

  python tools/sweep_attn.py > gpurun_out/attn_sweep.txt
Env knobs are read per launch plan, so one process sweeps them all."""
import os
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2511_16665_b200.engine import Engine  # noqa: E402

SHAPES = [(1, 1024, 1), (8, 1024, 1), (32, 1024, 1), (64, 1024, 1), (1, 1024, 65), (1, 1024, 17), (5, 700, 49),
          (8, 1024, 33), (16, 700, 17), (31, 700, 17), (31, 2000, 17), (4, 700, 9)]
TREE = [("148", "256"), ("296", "256"), ("148", "128"), ("296", "128"), ("592", "64"), ("74", "256"),
        ("592", "128"), ("296", "64"), ("1184", "64")]
if "--tree-only" in sys.argv:  # the tcgen05 tree kernel's split plan only
    SHAPES = [s for s in SHAPES if s[2] * 7 > 16]
DEC = [("296", "256"), ("592", "128"), ("1184", "64")]
if "--dec-only" in sys.argv:  # decode split targets at the AR-phase batch sizes
    SHAPES = [(32, 1024, 1), (48, 1500, 1), (64, 1024, 1), (64, 2048, 1)]
    DEC = [("296", "256"), ("444", "256"), ("592", "256"), ("888", "256"), ("592", "512"), ("148", "256")]

eng = Engine("qwen2.5-7b", max_slots=64, max_ctx=2400)


def probe(b, ctx, r):
    ms, by = eng.probe_attention(b, ctx, r, 56)
    return ms * 1e3, by / ms / 1e6


for b, ctx, r in SHAPES:
    G = 7
    if r * G <= 16:
        for ctas, mc in DEC:
            os.environ["TLT_ATTN_DEC_CTAS"], os.environ["TLT_ATTN_DEC_MIN_CHUNK"] = ctas, mc
            us, gbs = probe(b, ctx, r)
            print(f"dec  b={b} ctx={ctx} rows={r} ctas={ctas} min={mc}: {us:.1f} us {gbs:.0f} GB/s", flush=True)
        os.environ.pop("TLT_ATTN_DEC_CTAS"), os.environ.pop("TLT_ATTN_DEC_MIN_CHUNK")
        continue
    os.environ["TLT_ATTN_TREE_DYN"] = "0"
    us, gbs = probe(b, ctx, r)
    print(f"tree b={b} ctx={ctx} rows={r} fixed-256 (r1): {us:.1f} us {gbs:.0f} GB/s", flush=True)
    os.environ["TLT_ATTN_TREE_DYN"] = "1"
    for ctas, mc in TREE:
        os.environ["TLT_ATTN_TREE_CTAS"], os.environ["TLT_ATTN_TREE_MIN_CHUNK"] = ctas, mc
        us, gbs = probe(b, ctx, r)
        print(f"tree b={b} ctx={ctx} rows={r} ctas={ctas} min={mc}: {us:.1f} us {gbs:.0f} GB/s", flush=True)
    os.environ.pop("TLT_ATTN_TREE_CTAS"), os.environ.pop("TLT_ATTN_TREE_MIN_CHUNK")
eng.close()
