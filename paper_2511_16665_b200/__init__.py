"""B200-native TLT adaptive speculative-decoding rollout step (arXiv 2511.16665).

Host mirror of the reference ``specsim`` hot path over the C-ABI in
``include/tlt_b200.h``; kernels live in ``csrc/`` (sm_100a).
"""
from ._lib import lib, LIB_PATH, TltError  # noqa: F401
