"""Flash-decode attention split sweep: tlt_probe_attention at (b, ctx) for the
TLT_ATTN_DEC_CTAS target set in the environment (one process per setting)."""
import os
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2511_16665_b200.engine import Engine  # noqa: E402

eng = Engine("qwen2.5-7b", max_slots=64, max_ctx=2304)
for b, ctx in [(1, 256), (1, 300), (1, 512), (4, 256), (1, 1024), (4, 1024), (16, 1024), (32, 1024), (64, 1024), (32, 2048), (8, 2048)]:
    ms, by = eng.probe_attention(b, ctx, 1, 56)
    print(f"ctas={os.environ.get('TLT_ATTN_DEC_CTAS', 'default')} b={b} ctx={ctx} us={ms * 1e3:.1f} "
          f"GB/s={by / ms / 1e6:.0f}", flush=True)
eng.close()
