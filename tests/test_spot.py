"""Spot drafter training (reference data_buffer.hpp,
packing.hpp, spot_trainer.hpp, checkpoint.hpp).

CPU: DataBuffer eviction / budgeted sampling and pack_sequences are checked
against the UNMODIFIED reference (oracle/_ref) on random sequences; FNV-1a-64
against the reference; checkpoint round trip and every corruption check.
GPU: the torch drafter used by the trainer reproduces the engine's drafter
rows; training on the target's own rollouts (C2 export) lowers the loss and
raises the mean accept length of a held-out rollout, which stays lossless;
a checkpoint restores bit-identical drafter weights into a fresh engine."""
import ctypes as C
import random

import numpy as np
import pytest

import oracle as O
from paper_2511_16665_b200 import spot as S

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference bridge not built")


def _ref():
    R = O.ref()
    R.ref_databuf_create.restype = C.c_void_p
    R.ref_databuf_create.argtypes = [C.c_longlong]
    R.ref_databuf_destroy.argtypes = [C.c_void_p]
    R.ref_databuf_insert.argtypes = [C.c_void_p, C.c_longlong, C.c_void_p, C.c_void_p, C.c_int]
    R.ref_databuf_size.argtypes = [C.c_void_p]
    R.ref_databuf_sample.argtypes = [C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p, C.c_void_p, C.c_int,
                                     C.c_longlong]
    R.ref_pack.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_longlong, C.c_void_p, C.c_int, C.c_void_p,
                           C.c_longlong]
    R.ref_fnv1a64.restype = C.c_ulonglong
    R.ref_fnv1a64.argtypes = [C.c_char_p, C.c_ulonglong]
    return R


def _flat(seqs):
    toks = np.asarray([t for s in seqs for t in s] or [0], np.int32)
    lens = np.asarray([len(s) for s in seqs] or [0], np.int32)
    return toks, lens


@needs_ref
@pytest.mark.parametrize("seed,retention", [(0, 1), (1, 0), (2, 2), (3, 1)])
def test_data_buffer_matches_reference(seed, retention):
    R = _ref()
    g = random.Random(seed)
    h = R.ref_databuf_create(retention)
    buf = S.DataBuffer(retention)
    try:
        step = 0
        for it in range(30):
            step += g.choice([0, 0, 1])
            seqs = [[g.randrange(50) for _ in range(g.choice([0, 1, 3, 7, 7, 12, 30]))] for _ in range(g.randrange(0, 6))]
            t, l = _flat(seqs)
            R.ref_databuf_insert(h, step, t.ctypes.data, l.ctypes.data, len(seqs))
            buf.insert(step, seqs)
            assert R.ref_databuf_size(h) == len(buf.entries)
            for cur in (step, step + 1):
                budget = g.choice([1, 5, 20, 60, 500])
                ot = np.zeros(4096, np.int32)
                ol = np.zeros(512, np.int32)
                n = R.ref_databuf_sample(h, cur, budget, ot.ctypes.data, ol.ctypes.data, 512, 4096)
                assert n >= 0
                ref, off = [], 0
                for i in range(n):
                    ref.append(ot[off:off + ol[i]].tolist())
                    off += ol[i]
                assert [e.tokens for e in buf.sample(cur, budget)] == ref
    finally:
        R.ref_databuf_destroy(h)


@needs_ref
@pytest.mark.parametrize("seed,capacity", [(0, 8), (1, 16), (2, 5), (3, 64), (4, 1)])
def test_pack_sequences_matches_reference(seed, capacity):
    R = _ref()
    g = random.Random(seed)
    for _ in range(20):
        seqs = [[g.randrange(100) for _ in range(g.choice([0, 1, 2, 5, 8, 9, 16, 40]))] for _ in range(g.randrange(0, 12))]
        t, l = _flat(seqs)
        bounds = np.zeros(1024, np.int32)
        otok = np.zeros(8192, np.int32)
        nb = R.ref_pack(t.ctypes.data, l.ctypes.data, len(seqs), capacity, bounds.ctypes.data, 1024,
                        otok.ctypes.data, 8192)
        assert nb >= 0
        ref_b, cur = [], []
        for b in bounds[:nb]:
            if b < 0:
                ref_b.append(cur)
                cur = []
            else:
                cur.append(int(b))
        p = S.pack_sequences([len(s) for s in seqs], capacity)
        assert p.boundaries == ref_b
        mine = [t for pack in p.packs for (i, n) in pack for t in seqs[i][:n]]
        assert mine == otok[:len(mine)].tolist() and len(mine) == sum(sum(b) for b in ref_b)


@needs_ref
def test_fnv1a64_matches_reference():
    R = _ref()
    for data in [b"", b"a", b"foobar", bytes(range(256)) * 3]:
        assert S._fnv_np(data) == S.fnv1a64(data) == R.ref_fnv1a64(data, len(data))
    assert S.fnv1a64(b"a") == 0xaf63dc4c8601ec8c


def test_checkpoint_round_trip_and_corruption():
    rng = np.random.default_rng(0)
    shape = dict(vocab=64, hidden=16, layers=2, heads=4, kv_heads=2, head_dim=4, ffn=24)
    tens = {"fc": rng.integers(0, 65535, (16, 32)).astype(np.uint16),
            "qkv": rng.integers(0, 65535, (32, 16)).astype(np.uint16)}
    b = S.checkpoint_bytes(7, shape, tens)
    ver, sh, got = S.checkpoint_from_bytes(b)
    assert ver == 7 and sh == shape and all(np.array_equal(got[k], tens[k]) for k in tens)
    with pytest.raises(S.CheckpointError, match="checksum"):
        bad = bytearray(b)
        bad[len(bad) // 2] ^= 0x40
        S.checkpoint_from_bytes(bytes(bad))
    with pytest.raises(S.CheckpointError, match="truncated"):
        S.checkpoint_from_bytes(b[:10])
    body = bytearray(b[:-8])
    body[0:8] = b"XXXXXXXX"
    with pytest.raises(S.CheckpointError, match="bad magic"):
        S.checkpoint_from_bytes(bytes(body) + S.struct.pack("<Q", S.fnv1a64(bytes(body))))
    body = bytearray(b[:-8]) + b"\x00"
    with pytest.raises(S.CheckpointError, match="trailing"):
        S.checkpoint_from_bytes(bytes(body) + S.struct.pack("<Q", S.fnv1a64(bytes(body))))


# ------------------------------------------------------------------- GPU
def _collect(eng, prompts, max_lens):
    """Greedy rollout of the target; C2 export of every finished request."""
    res = eng.run_rollout(prompts, max_lens, enable_sd=False, keep_finished=True)
    out = []
    for i in range(len(prompts)):
        toks, feats = eng.export_sequence(i)
        out.append((toks.tolist(), feats))
        eng.release(i)
    return res, out


@pytest.mark.gpu
def test_gpu_torch_drafter_matches_engine_rows():
    import torch
    from paper_2511_16665_b200.engine import Engine
    eng = Engine("tiny", max_slots=2, max_ctx=256)
    rng = np.random.default_rng(1)
    prompts = [rng.integers(2, 4096, 20).tolist() for _ in range(2)]
    _, samples = _collect(eng, prompts, [24, 24])
    tr = S.DrafterTrainer(eng)
    eng.set_debug(True)
    for i, (toks, feats) in enumerate(samples):
        eng.prefill([0], [toks[:-1]])  # committed = toks[:-2], root = toks[-2]
        r = eng.sd_step((2, 2, 2), [0])
        row = dict(eng.debug_expansions(0))[()]
        n = len(toks) - 1   # rows 0..n-1: inputs (feature_{r-1}, tok_r); row n-1 is the root
        dev = tr.params["fc"].device
        t = torch.as_tensor(toks[:n], device=dev)
        f = torch.cat([torch.zeros((1, eng.hidden), device=dev, dtype=torch.bfloat16), feats[:n - 1].to(dev)], 0)
        with torch.no_grad():
            logits = tr.forward(t, f, torch.arange(n, device=dev), torch.zeros(n, device=dev, dtype=torch.int64))
        p = torch.softmax(logits[-1].double(), -1).cpu().numpy()
        m = row > 1e-4
        assert np.abs(np.log(p[m]) - np.log(row[m])).max() < 0.2
        assert int(np.argmax(p)) == int(np.argmax(row))
        eng.release(0)
    eng.close()


@pytest.mark.gpu
def test_gpu_spot_training_improves_acceptance_and_checkpoint_restores(tmp_path):
    import torch
    from paper_2511_16665_b200.engine import Engine
    eng = Engine("tiny", max_slots=16, max_ctx=512, init={"fc_noise": 0.6})  # a weak initial drafter
    rng = np.random.default_rng(7)
    train_prompts = [rng.integers(2, 4096, 16).tolist() for _ in range(32)]
    test_prompts = [rng.integers(2, 4096, 16).tolist() for _ in range(8)]
    strat = (6, 4, 24)

    def accept(prompts):
        r = eng.run_rollout(prompts, [96] * len(prompts), enable_sd=True, elastic_threshold=64, strategy=strat)
        return r["accepted_total"] / r["verify_events"], r["tokens"]

    before, _ = accept(test_prompts)
    buf = S.DataBuffer(retention=1)
    for step in range(2):
        _, samples = _collect(eng, train_prompts[16 * step:16 * step + 16], [160] * 16)
        buf.insert(step, [s[0] for s in samples], [s[1] for s in samples])
    tr = S.DrafterTrainer(eng, lr=1e-3)
    cfg = S.SpotTrainConfig(current_step=1, token_budget=8192, pack_capacity=1024)
    ck = str(tmp_path / "drafter.ckpt")
    log = S.spot_train_loop(tr, buf, cfg, iterations=60, checkpoint_path=ck)
    assert log.iterations == 60 and log.versions[-1] == 60 and S.drafter_version(eng) == 60
    assert np.mean(log.losses[-5:]) < 0.7 * np.mean(log.losses[:3]), (log.losses[:3], log.losses[-5:])
    after, toks_after = accept(test_prompts)
    assert after > before, (before, after)
    ar = eng.run_rollout(test_prompts, [96] * 8, enable_sd=False)
    from parity_util import greedy_streams_agree, tiny_oracle_model
    m = tiny_oracle_model()
    try:
        for p, a, b in zip(test_prompts, toks_after, ar["tokens"]):
            ok, k, margin = greedy_streams_agree(m, p, a, b, 4096)
            assert ok, (k, margin)
    finally:
        O.orc().orc_model_destroy(m)
    # checkpoint -> fresh engine: bit-identical trainable tensors, same version
    fresh = Engine("tiny", max_slots=2, max_ctx=128, init={"fc_noise": 0.6})
    assert S.restore_checkpoint(fresh, open(ck, "rb").read()) == 60
    a, b = S.drafter_tensors(eng), S.drafter_tensors(fresh)
    for k, (t, trainable) in a.items():
        if trainable:
            assert torch.equal(t.view(torch.int16), b[k][0].view(torch.int16)), k
    fresh.close()
    eng.close()
