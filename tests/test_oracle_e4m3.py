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


def test_oracle_fp8_drafter_head_close_to_bf16():
    """The oracle's e4m3 drafter LM head (drafter_lm_fp8) changes the drafter
    rows only by quantisation noise: same top tokens on the tiny model, log
    probabilities of the likely tokens within 0.5, and not bit-identical."""
    from paper_2511_16665_b200.engine import INITS, MODELS

    L = O.orc()
    T, I = MODELS["tiny"], INITS["tiny"]
    cfg = O.ModelCfg(T["vocab"], T["hidden"], T["layers"], T["heads"], T["kv_heads"], T["head_dim"], T["ffn"],
                     T["qkv_bias"], T["rope_theta"], T["rms_eps"], 256)
    rows = []
    for fp8 in (0, 1):
        ini = O.InitCfg(I["seed"], I["layer_scale"], I["lm_gain"], I["lm_alt"], I["lm_noise"], I["fc_noise"], fp8)
        m = L.orc_model_create(C.byref(cfg), C.byref(ini), 4)
        assert m
        s = L.orc_seq_create(m)
        prompt = (C.c_int32 * 12)(*range(5, 17))
        L.orc_seq_append.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
        assert L.orc_seq_append(s, prompt, 12) == 0
        p = np.zeros(T["vocab"], np.float64)
        path = (C.c_int32 * 1)(0)
        L.orc_drafter_row.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        assert L.orc_drafter_row(s, path, 0, p.ctypes.data_as(C.c_void_p), None) == 0
        rows.append(p)
        L.orc_seq_destroy(s)
        L.orc_model_destroy(m)
    a, b = rows
    assert not np.array_equal(a, b)
    assert np.argmax(a) == np.argmax(b)
    likely = a > 1e-3
    assert np.abs(np.log(a[likely]) - np.log(b[likely])).max() < 0.5
