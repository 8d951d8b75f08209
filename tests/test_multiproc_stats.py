"""C1 on CPU: world_size-2 gloo all-gather of per-rank BEG-MAB records, applied
in rank order to every replica. All replicas must end
bit-identical; with one rank the merge reduces to the local beg_record
sequence (beg_mab.hpp:111-134)."""
import os
import random

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ARMS = [(10, 8, 64), (6, 8, 64), (10, 8, 48), (6, 8, 48), (10, 8, 32), (6, 8, 32), (10, 8, 16), (6, 8, 16)]
THR = [1, 2, 8, 16]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_16665_b200.engine import Mab, Rng
    mab = Mab(ARMS, THR, 0.1, 20)
    rng = Rng(1234, 0x53454C + rank)
    g = random.Random(rank)
    for step in range(40):
        batch = g.choice([1, 3, 9, 20])
        arm, s = mab.select(batch, rng)
        lens = [g.randrange(0, s[0] + 1) for _ in range(batch)]
        elapsed = 1.0 + g.random()
        a_bar = sum(lens) / batch + 1.0
        reward = a_bar * batch / elapsed
        rec = torch.tensor([float(arm), reward, a_bar], dtype=torch.float64)
        out = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, rec)
        for r in range(world):  # rank order: every replica applies the same sequence
            mab.apply_record(int(out[r][0].item()), out[r][1].item(), out[r][2].item())
    # reward windows (median, fill) must agree; selection counts are local decisions
    stats = torch.tensor([v for i in range(len(ARMS)) for v in (mab.arm_stats(i)[0], mab.arm_stats(i)[2])],
                         dtype=torch.float64)
    gathered = [torch.zeros_like(stats) for _ in range(world)]
    dist.all_gather(gathered, stats)
    q.put((rank, all(torch.equal(gathered[0], t) for t in gathered)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_allgather_merge_keeps_replicas_identical(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.randrange(1000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def _rollout_worker(rank, world, port, q, use_lib=False):
    """bench.py's C1 path: per 'rollout' each rank records into its local
    replica, then merge_bandit_stats all-gathers the logs and applies them in
    rank order to the shared replica; shared replicas must be bit-identical
    and equal to one sequential application of rank 0's then rank 1's records."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_16665_b200.engine import C1, Mab, Rng, merge_bandit_stats
    local, shared = Mab(ARMS, THR, 0.1, 20), Mab(ARMS, THR, 0.1, 20)
    c1 = C1.from_dist(dist) if use_lib else None  # C1 inside the library (tlt_c1_merge)
    rng = Rng(99, 0x53454C + rank)
    g = random.Random(7 + rank)
    total = 0
    all_logs = []
    for rollout in range(3):
        mine = []
        for step in range(10 + rank):  # ranks run different numbers of SD steps
            batch = g.choice([1, 4, 12, 25])
            arm, s = local.select(batch, rng)
            lens = [g.randrange(0, s[0] + 1) for _ in range(batch)]
            local.record(s, 1.0 + g.random(), lens)
        total += merge_bandit_stats(dist, local, shared, c1)
    stats = torch.tensor([v for i in range(len(ARMS)) for v in (shared.arm_stats(i)[0], shared.arm_stats(i)[2])],
                         dtype=torch.float64)
    gathered = [torch.zeros_like(stats) for _ in range(world)]
    dist.all_gather(gathered, stats)
    local_stats = torch.tensor([v for i in range(len(ARMS)) for v in (local.arm_stats(i)[0], local.arm_stats(i)[2])],
                               dtype=torch.float64)
    ok = all(torch.equal(gathered[0], t) for t in gathered) and torch.equal(local_stats, stats)
    ok = ok and total == 3 * sum(10 + r for r in range(world))
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("use_lib", [False, True])
def test_gloo_rollout_boundary_merge(use_lib):
    """use_lib: the library's C1 (fixed-size record blocks, rank-order apply in
    C++) over a host all-gather callback on the gloo group."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.randrange(1000, 2000)
    procs = [ctx.Process(target=_rollout_worker, args=(r, world, port, q, use_lib)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


@pytest.mark.gpu
def test_gpu_c1_nccl_world1_equals_local_sequence():
    """C1 over NCCL inside the library, one rank: the shared replica equals a
    replica that ran the same beg_record sequence locally."""
    from paper_2511_16665_b200.engine import C1, Engine, Mab, Rng
    eng = Engine("tiny", max_slots=2, max_ctx=64)
    c1 = C1.nccl(eng, C1.nccl_unique_id(), 1, 0)
    local, shared, ref = Mab(ARMS, THR, 0.1, 20), Mab(ARMS, THR, 0.1, 20), Mab(ARMS, THR, 0.1, 20)
    rng, rref = Rng(5, 1), Rng(5, 1)
    g = random.Random(3)
    for rollout in range(4):
        for step in range(15):
            batch = g.choice([1, 4, 12, 25])
            _, s = local.select(batch, rng)
            _, s2 = ref.select(batch, rref)
            assert s == s2
            lens = [g.randrange(0, s[0] + 1) for _ in range(batch)]
            el = 1.0 + g.random()
            local.record(s, el, lens)
            ref.record(s, el, lens)
        assert c1.merge(local, shared) == 15
        for i in range(len(ARMS)):
            assert shared.arm_stats(i)[0] == ref.arm_stats(i)[0] and shared.arm_stats(i)[2] == ref.arm_stats(i)[2]
            assert shared.arm_window(i) == ref.arm_window(i) == local.arm_window(i)
    del c1
    eng.close()
