"""The oracle's e4m3 row quantisation (orc_e4m3_quant_row, emulating the
engine's k_quant_rows_e4m3: scale = amax / 448, RNE saturating e4m3 of
x / scale) against torch's float8_e4m3fn cast -- the same chain the GPU test
test_gpu_gemm_e4m3.py closes from the other side (GPU == torch)."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle as O


@pytest.mark.parametrize("seed,scale", [(0, 1.0), (1, 1e-3), (2, 37.0), (3, 1e-6)])
def test_e4m3_quant_row_matches_torch(seed, scale):
    L = O.orc()
    L.orc_e4m3_quant_row.restype = C.c_float
    L.orc_e4m3_quant_row.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    rng = np.random.default_rng(seed)
    for n in (1, 7, 3584):
        x = (rng.standard_normal(n) * scale).astype(np.float32)
        x[::5] *= 1e-4  # deep subnormal range of e4m3 after scaling
        if n > 10:
            x[3] = 0.0
        # bf16-representable inputs, as the engine quantises bf16 rows
        x = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
        q = np.zeros(n, np.float32)
        s = L.orc_e4m3_quant_row(x.ctypes.data_as(C.c_void_p), n, q.ctypes.data_as(C.c_void_p))
        amax = np.float32(np.abs(x).max())
        s_ref = np.float32(amax / np.float32(448.0)) if amax > 0 else np.float32(1.0)
        assert np.float32(s) == s_ref
        q_ref = (torch.from_numpy(x) / torch.tensor(s_ref)).to(torch.float8_e4m3fn).float().numpy()
        assert np.array_equal(q, q_ref), np.flatnonzero(q != q_ref)[:5]


def test_e4m3_zero_row():
    L = O.orc()
    L.orc_e4m3_quant_row.restype = C.c_float
    L.orc_e4m3_quant_row.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    x = np.zeros(16, np.float32)
    q = np.ones(16, np.float32)
    assert L.orc_e4m3_quant_row(x.ctypes.data_as(C.c_void_p), 16, q.ctypes.data_as(C.c_void_p)) == 1.0
    assert not q.any()
