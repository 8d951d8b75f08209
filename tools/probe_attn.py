"""Engine attention probes (tlt_probe_attention): b:ctx:rows ..."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2511_16665_b200.engine import Engine  # noqa: E402

eng = Engine("qwen2.5-7b", max_slots=64, max_ctx=2400)
for spec in sys.argv[1:]:
    b, ctx, r = (int(x) for x in spec.split(":"))
    ms, by = eng.probe_attention(b, ctx, r, 56)
    print(f"b={b} ctx={ctx} rows={r} us={ms * 1e3:.1f} GB/s={by / ms / 1e6:.0f}", flush=True)
eng.close()
