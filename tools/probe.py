"""Engine GEMM-site probes (tlt_probe_kernel) at given (kind, M) pairs: kind:M ..."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2511_16665_b200.engine import Engine  # noqa: E402

eng = Engine("qwen2.5-7b", max_slots=32, max_ctx=512)
for spec in sys.argv[1:]:
    kind, m = (int(x) for x in spec.split(":"))
    ms, b, f = eng.probe_kernel(kind, m, 56)
    print(f"kind={kind} M={m} us={ms * 1e3:.1f} GB/s={b / ms / 1e6:.0f} TF/s={f / ms / 1e9:.0f}", flush=True)
eng.close()
