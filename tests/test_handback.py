"""C2: drafter training samples handed back to the trainer
rank. CPU: world-size-2 gloo exchange of synthetic (tokens, bf16 features)
sequences, received bit-exact in rank order. GPU: tlt_export_sequence returns
the slot's committed token stream (prompt + emitted) and its target features."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _samples(rank):
    g = torch.Generator().manual_seed(100 + rank)
    out = []
    for k in range(2 + rank):
        L = 3 + 5 * k + rank
        toks = torch.randint(0, 4096, (L + 1,), generator=g, dtype=torch.int32).numpy()
        feats = torch.randn((L, 16), generator=g).to(torch.bfloat16)
        out.append((toks, feats))
    return out


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_16665_b200.engine import handback_samples
    got = handback_samples(dist, _samples(rank), trainer_rank=0)
    if rank == 0:
        want = [(r, t, f) for r in range(world) for t, f in _samples(r)]
        ok = len(got) == len(want) and all(
            gr == wr and np.array_equal(gt.numpy(), wt) and torch.equal(gf.view(torch.int16), wf.view(torch.int16))
            for (gr, gt, gf), (wr, wt, wf) in zip(got, want))
        q.put(("trainer", ok, len(got)))
    else:
        q.put(("worker", got == [], 0))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_handback_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(60)
    assert all(p.exitcode == 0 for p in ps)
    assert all(ok for _, ok, _ in res), res
    assert sum(n for _, _, n in res) == 2 + 3


@pytest.mark.gpu
def test_gpu_export_sequence():
    from paper_2511_16665_b200.engine import Engine
    V = 4096
    rng = np.random.default_rng(2)
    prompts = [rng.integers(2, V, 16).tolist() for _ in range(2)]
    eng = Engine("tiny", max_slots=2, max_ctx=256, device=0)
    eng.prefill([0, 1], prompts)
    emitted = [[], []]
    for _ in range(3):
        r = eng.sd_step((4, 4, 16), [0, 1])
        for i in range(2):
            emitted[i] += r.accepted[i] + [int(r.bonus[i])]
    toks, _ = eng.ar_step([0, 1])
    for i in range(2):
        emitted[i].append(int(toks[i]))
    for i in range(2):
        t, f = eng.export_sequence(i)
        L = eng.slot_len(i)
        assert t.tolist() == prompts[i] + emitted[i]
        assert len(t) == L + 1 and tuple(f.shape) == (L, eng.hidden) and f.is_cuda
        ff = f.float()
        assert torch.isfinite(ff).all() and ff.abs().sum(dim=1).min().item() > 0
        tc, fc = eng.export_sequence(i, device=False)
        assert np.array_equal(tc, t) and torch.equal(fc.view(torch.int16), f.cpu().view(torch.int16))
    eng.close()


@pytest.mark.gpu
def test_gpu_handback_of_exported_cuda_tensors_over_gloo():
    """samples exported as CUDA tensors travel over a gloo group
    (CPU transport) — world size 1, the trainer rank gets them back on CPU."""
    from torch.distributed import FileStore

    from paper_2511_16665_b200.engine import Engine, handback_samples
    import tempfile
    rng = np.random.default_rng(3)
    prompts = [rng.integers(2, 4096, 12).tolist() for _ in range(2)]
    eng = Engine("tiny", max_slots=2, max_ctx=256, device=0)
    eng.run_rollout(prompts, [10, 15], enable_sd=True, elastic_threshold=8, strategy=(4, 4, 16), keep_finished=True)
    samples = [eng.export_sequence(i) for i in range(2)]
    with tempfile.NamedTemporaryFile() as f:
        dist.init_process_group("gloo", store=FileStore(f.name, 1), rank=0, world_size=1)
        try:
            got = handback_samples(dist, samples, trainer_rank=0)
        finally:
            dist.destroy_process_group()
    assert len(got) == 2
    for (r, t, feats), (wt, wf) in zip(got, samples):
        assert r == 0 and not feats.is_cuda and t.tolist() == wt.tolist()
        assert torch.equal(feats.view(torch.int16), wf.cpu().view(torch.int16))
    eng.close()
