"""Spot drafter training on the GPU.

The reference trains its count drafter on idle workers: rollout sequences go
into a DataBuffer (data_buffer.hpp:48-68), a budgeted sample is packed
(packing.hpp:30-61) and trained for a number of iterations (spot_train_loop,
spot_trainer.hpp:42-64) with checkpoints (checkpoint.hpp:90-209) and the
result is published as the rollout's DrafterSnapshot (rollout.hpp:61-64).
Here the drafter is the engine's one-layer EAGLE model, so:

* DataBuffer / pack_sequences restate the reference semantics exactly
  (retention eviction, previous-step-longest-first budgeted sampling,
  first-fit-decreasing packing without padding, truncation at capacity) over
  C2 samples (tokens + the target's bf16 features, tlt_export_sequence);
* train_on_batch runs the drafter forward in torch on the engine's own weight
  buffers (tlt_drafter_tensors: the same math as the engine's drafter row —
  x = [feature_{t-1} || E[tok_t]] W_fc^T, one decoder layer with interleaved
  RoPE / GQA / SwiGLU, the shared final norm + LM head) with causal attention
  inside each packed sequence, loss = cross entropy of the next token, AdamW
  on fp32 master copies of the trainable tensors (fc + the layer); the shared
  embedding / final norm / LM head stay frozen;
* publish writes the bf16 weights back in place and calls
  tlt_drafter_published (drafter KV of live slots is recomputed on their next
  EAGLE step; captured CUDA graphs keep pointing at the same buffers);
* checkpoints ("TLTDCKP1": magic, byte-order marker, format version, drafter
  version, model shape, named bf16 tensors, FNV-1a-64 trailer — the
  reference's SSDCKPT1 scheme, checkpoint.hpp:16-22, 90-158, for the neural
  drafter) restore bit-identical weights; corrupt files raise; snapshot-
  isolated asynchronous save (checkpoint.hpp:204-209).
"""
from __future__ import annotations

import ctypes as C
import math
import struct
import threading
from dataclasses import dataclass, field

import numpy as np

from .engine import Engine, _check
from ._lib import lib


class CheckpointError(RuntimeError):
    """Reference CheckpointError (errors.hpp)."""


# ------------------------------------------------------------------ DataBuffer
@dataclass
class DataBufferEntry:
    step_id: int
    tokens: list
    features: object = None  # torch bf16 [len(tokens) - 1][d] (C2 payload), optional

    def length(self):
        return len(self.tokens)


class DataBuffer:
    """data_buffer.hpp:25-73: entries older than current_step - retention are
    evicted on insert; sample() takes the previous step's entries by
    descending length, then the current step's, each pass stopping at the
    first entry that would overflow the token budget (stable order)."""

    def __init__(self, retention: int = 1):
        if retention < 0:
            raise ValueError("retention: must be >= 0")
        self.retention = retention
        self.current_step = 0
        self.entries: list[DataBufferEntry] = []

    def insert(self, step_id: int, sequences, features=None):
        self.current_step = max(self.current_step, step_id)
        for i, s in enumerate(sequences):
            self.entries.append(DataBufferEntry(step_id, list(s), None if features is None else features[i]))
        self.entries = [e for e in self.entries if not e.step_id < self.current_step - self.retention]

    def sample(self, current_step: int, token_budget: int):
        if token_budget < 1:
            raise ValueError("token_budget: must be >= 1")
        out, used = [], 0
        for step in (current_step - 1, current_step):
            pool = [e for e in self.entries if e.step_id == step]
            pool.sort(key=lambda e: -e.length())  # list.sort is stable, like std::stable_sort
            for e in pool:
                if used + e.length() > token_budget:
                    break
                out.append(e)
                used += e.length()
        return out


# ------------------------------------------------------------------ packing
@dataclass
class PackedBatch:
    packs: list = field(default_factory=list)        # [pack][(entry index, length)] in placement order
    boundaries: list = field(default_factory=list)   # [pack][member lengths]
    capacity: int = 0

    def total_tokens(self):
        return sum(sum(b) for b in self.boundaries)


def pack_sequences(lengths, capacity: int) -> PackedBatch:
    """packing.hpp:30-61: first-fit-decreasing over min(len, capacity)
    (stable for equal lengths), empty sequences skipped, sequences longer than
    capacity truncated (suffix dropped). Returns member (index, length) lists."""
    if capacity == 0:
        raise ValueError("capacity: must be >= 1")
    idx = sorted(range(len(lengths)), key=lambda i: -min(lengths[i], capacity))
    out = PackedBatch(capacity=capacity)
    free = []
    for i in idx:
        n = min(lengths[i], capacity)
        if n == 0:
            continue
        slot = next((s for s in range(len(free)) if free[s] >= n), len(out.packs))
        if slot == len(out.packs):
            out.packs.append([])
            out.boundaries.append([])
            free.append(capacity)
        out.packs[slot].append((i, n))
        out.boundaries[slot].append(n)
        free[slot] -= n
    return out


# ------------------------------------------------------------------ checkpoint
MAGIC = b"TLTDCKP1"
BYTE_ORDER = 0x01020304
FORMAT_VERSION = 1


def fnv1a64(data: bytes) -> int:
    """checkpoint.hpp:26-33."""
    h = 0xcbf29ce484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def _fnv_np(data: bytes) -> int:
    """FNV-1a-64 of a (possibly GB-sized) blob, computed by the library (tlt_fnv1a64)."""
    L = lib()
    L.tlt_fnv1a64.restype = C.c_uint64
    L.tlt_fnv1a64.argtypes = [C.c_char_p, C.c_size_t]
    return L.tlt_fnv1a64(data, len(data))


def checkpoint_bytes(version: int, shape: dict, tensors: dict) -> bytes:
    """name -> bf16 bits (np.uint16 [rows][cols]); little-endian throughout."""
    w = bytearray(MAGIC)
    w += struct.pack("<IIq", BYTE_ORDER, FORMAT_VERSION, version)
    w += struct.pack("<7i", *(shape[k] for k in ("vocab", "hidden", "layers", "heads", "kv_heads", "head_dim", "ffn")))
    w += struct.pack("<Q", len(tensors))
    for name, arr in tensors.items():
        nb = name.encode()
        a = np.ascontiguousarray(arr, dtype="<u2")
        w += struct.pack("<I", len(nb)) + nb + struct.pack("<qq", a.shape[0], a.shape[1]) + a.tobytes()
    w += struct.pack("<Q", _fnv_np(bytes(w)))
    return bytes(w)


def checkpoint_from_bytes(data: bytes):
    """checkpoint.hpp:116-158 checks: size, checksum, magic, byte order,
    format version, shapes, trailing bytes."""
    if len(data) < len(MAGIC) + 8:
        raise CheckpointError("corrupt checkpoint: truncated")
    (stored,) = struct.unpack("<Q", data[-8:])
    if stored != _fnv_np(data[:-8]):
        raise CheckpointError("corrupt checkpoint: checksum mismatch")
    body, pos = data[:-8], 0

    def take(n):
        nonlocal pos
        if pos + n > len(body):
            raise CheckpointError("corrupt checkpoint: truncated")
        b = body[pos:pos + n]
        pos += n
        return b

    if take(8) != MAGIC:
        raise CheckpointError("corrupt checkpoint: bad magic")
    bo, fv, version = struct.unpack("<IIq", take(16))
    if bo != BYTE_ORDER:
        raise CheckpointError("corrupt checkpoint: byte-order mismatch")
    if fv != FORMAT_VERSION:
        raise CheckpointError("corrupt checkpoint: format version mismatch")
    shape = dict(zip(("vocab", "hidden", "layers", "heads", "kv_heads", "head_dim", "ffn"), struct.unpack("<7i", take(28))))
    (n,) = struct.unpack("<Q", take(8))
    tensors = {}
    for _ in range(n):
        (ln,) = struct.unpack("<I", take(4))
        name = take(ln).decode()
        rows, cols = struct.unpack("<qq", take(16))
        if rows < 0 or cols < 0:
            raise CheckpointError("corrupt checkpoint: invalid tensor shape")
        tensors[name] = np.frombuffer(take(2 * rows * cols), dtype="<u2").reshape(rows, cols).copy()
    if pos != len(body):
        raise CheckpointError("corrupt checkpoint: trailing bytes")
    return version, shape, tensors


# ------------------------------------------------------------------ engine weights
class TensorView(C.Structure):
    _fields_ = [("name", C.c_char_p), ("ptr", C.c_void_p), ("rows", C.c_int64), ("cols", C.c_int64),
                ("trainable", C.c_int32)]


class _CAI:
    """__cuda_array_interface__ over an engine buffer (bf16 as int16 bits)."""

    def __init__(self, ptr, rows, cols):
        self.__cuda_array_interface__ = {"shape": (int(rows), int(cols)), "typestr": "<i2",
                                         "data": (int(ptr), False), "version": 3}


def drafter_tensors(engine: Engine):
    """name -> (torch bf16 view of the engine buffer, trainable)."""
    import torch
    L = lib()
    n = C.c_int32()
    _check(L.tlt_drafter_tensors(engine.h, None, 0, C.byref(n)))
    arr = (TensorView * n.value)()
    _check(L.tlt_drafter_tensors(engine.h, arr, n.value, C.byref(n)))
    out = {}
    for v in arr:
        t = torch.as_tensor(_CAI(v.ptr, v.rows, v.cols), device=f"cuda:{engine.device}").view(torch.bfloat16)
        out[v.name.decode()] = (t, bool(v.trainable))
    return out


def save_checkpoint(engine: Engine, version: int | None = None) -> bytes:
    """Snapshot of the drafter's trainable tensors (bf16 bits) as TLTDCKP1 bytes."""
    import torch
    views = drafter_tensors(engine)
    if version is None:
        version = drafter_version(engine)
    tens = {k: t.view(torch.int16).cpu().numpy().view(np.uint16) for k, (t, tr) in views.items() if tr}
    m = engine.model
    return checkpoint_bytes(version, m, tens)


def save_checkpoint_async(engine: Engine, path: str, version: int | None = None) -> threading.Thread:
    """checkpoint.hpp:204-209: the state is copied at call time (device ->
    host snapshot), serialised and written off-thread."""
    import torch
    views = drafter_tensors(engine)
    ver = drafter_version(engine) if version is None else version
    snap = {k: t.view(torch.int16).cpu().numpy().view(np.uint16).copy() for k, (t, tr) in views.items() if tr}
    shape = dict(engine.model)

    def work():
        with open(path, "wb") as f:
            f.write(checkpoint_bytes(ver, shape, snap))

    th = threading.Thread(target=work, daemon=True)
    th.start()
    return th


def restore_checkpoint(engine: Engine, data: bytes):
    """Writes the checkpoint's tensors into the engine (bit-identical) and
    publishes them as the drafter snapshot of the checkpoint's version."""
    import torch
    version, shape, tensors = checkpoint_from_bytes(data)
    for k in ("vocab", "hidden", "layers", "heads", "kv_heads", "head_dim", "ffn"):
        if shape[k] != engine.model[k]:
            raise CheckpointError(f"checkpoint shape mismatch: {k}")
    views = drafter_tensors(engine)
    for name, bits in tensors.items():
        t, trainable = views.get(name, (None, False))
        if t is None or not trainable or tuple(t.shape) != bits.shape:
            raise CheckpointError(f"checkpoint tensor does not match the drafter: {name}")
        t.view(torch.int16).copy_(torch.from_numpy(bits.view(np.int16)).to(t.device))
    torch.cuda.synchronize(t.device)
    publish(engine, version)
    return version


def drafter_version(engine: Engine) -> int:
    v = C.c_int64()
    _check(lib().tlt_drafter_version(engine.h, C.byref(v)))
    return v.value


def publish(engine: Engine, version: int):
    _check(lib().tlt_drafter_published(engine.h, C.c_int64(version)))


# ------------------------------------------------------------------ trainer
@dataclass
class SpotTrainConfig:
    """spot_trainer.hpp:18-23 (+ optimiser knobs of the neural drafter)."""
    current_step: int = 0
    token_budget: int = 8192
    pack_capacity: int = 2048
    checkpoint_every: int = 50
    lr: float = 2e-4
    weight_decay: float = 0.0


@dataclass
class SpotTrainLog:
    iterations: int = 0
    versions: list = field(default_factory=list)
    losses: list = field(default_factory=list)
    preempted: bool = False
    checkpoints: int = 0


class DrafterTrainer:
    """The engine's EAGLE drafter in torch, on fp32 master copies of its
    trainable tensors; forward = the engine's drafter row (see module doc)."""

    def __init__(self, engine: Engine, lr=2e-4, weight_decay=0.0):
        import torch
        self.engine = engine
        self.m = engine.model
        self.views = drafter_tensors(engine)
        self.params = {k: torch.nn.Parameter(t.float().clone()) for k, (t, tr) in self.views.items() if tr}
        self.frozen = {k: t for k, (t, tr) in self.views.items() if not tr}
        self.opt = torch.optim.AdamW(self.params.values(), lr=lr, weight_decay=weight_decay, betas=(0.9, 0.95))
        hd = self.m["head_dim"]
        inv = torch.pow(torch.tensor(float(self.m["rope_theta"]), dtype=torch.float64),
                        -2.0 * torch.arange(hd // 2, dtype=torch.float64) / hd)
        self.inv_freq = inv.to(self.params["fc"].device)
        self.version = drafter_version(engine)

    def _rmsnorm(self, x, g):
        import torch
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + self.m["rms_eps"]) * g.float().view(-1)

    def _rope(self, x, pos):
        # interleaved (2i, 2i+1) pairs, angle = pos * theta^(-2i/hd) (engine / oracle table)
        import torch
        ang = pos.double()[:, None] * self.inv_freq[None, :]
        c, s = torch.cos(ang).float(), torch.sin(ang).float()
        x0, x1 = x[..., 0::2], x[..., 1::2]
        c, s = c[:, None, :], s[:, None, :]
        return torch.stack([x0 * c - x1 * s, x0 * s + x1 * c], dim=-1).flatten(-2)

    def forward(self, tokens, feats_prev, pos, seq_id):
        """tokens [N], feats_prev [N][d] (target feature of the previous
        position, 0 at a sequence start), pos [N], seq_id [N] (packed
        sequences attend causally within themselves). Returns logits [N][V]."""
        import torch
        import torch.nn.functional as F
        m, P, Fz = self.m, self.params, self.frozen
        d, H, KV, hd = m["hidden"], m["heads"], m["kv_heads"], m["head_dim"]
        emb = Fz["embed"][tokens].float()
        x = torch.cat([feats_prev.float(), emb], -1) @ P["fc"].t()
        h = self._rmsnorm(x, P["attn_norm"])
        qkv = h @ P["qkv"].t()
        if "qkv_bias" in P:
            qkv = qkv + P["qkv_bias"].view(-1)
        q = qkv[:, :H * hd].view(-1, H, hd)
        k = qkv[:, H * hd:(H + KV) * hd].view(-1, KV, hd)
        v = qkv[:, (H + KV) * hd:].view(-1, KV, hd)
        q, k = self._rope(q, pos), self._rope(k, pos)
        N = tokens.shape[0]
        idx = torch.arange(N, device=tokens.device)
        mask = (seq_id[:, None] == seq_id[None, :]) & (idx[None, :] <= idx[:, None])
        rep = H // KV
        att = F.scaled_dot_product_attention(q.transpose(0, 1), k.repeat_interleave(rep, 1).transpose(0, 1),
                                             v.repeat_interleave(rep, 1).transpose(0, 1), attn_mask=mask)
        x = x + att.transpose(0, 1).reshape(N, H * hd) @ P["o"].t()
        h = self._rmsnorm(x, P["mlp_norm"])
        gu = h @ P["gate_up"].t()
        a = F.silu(gu[:, 0::2]) * gu[:, 1::2]
        x = x + a @ P["down"].t()
        # the shared LM head stays bf16 (frozen); fp32 accumulation, fp32 logits
        return (self._rmsnorm(x, Fz["final_norm"]).to(torch.bfloat16) @ Fz["lm_head"].t()).float()

    def batch_from_pack(self, entries, pack):
        """One packed row: member sequences placed back to back (truncated to
        their packed length), inputs / labels / positions / sequence ids."""
        import torch
        dev = self.params["fc"].device
        d = self.m["hidden"]
        toks, feats, labels, pos, sid = [], [], [], [], []
        for j, (i, n) in enumerate(pack):
            e = entries[i]
            t = torch.as_tensor(np.asarray(e.tokens[:n], np.int64), device=dev)
            f = e.features[:n].to(dev) if e.features is not None else torch.zeros((n, d), device=dev,
                                                                                  dtype=torch.bfloat16)
            # row r: input (feature_{r-1}, tok_r), label tok_{r+1}; the last row has no label
            fp = torch.cat([torch.zeros((1, d), device=dev, dtype=f.dtype), f[:n - 1]], 0)
            lab = torch.cat([t[1:], torch.full((1,), -100, device=dev, dtype=torch.int64)])
            toks.append(t), feats.append(fp), labels.append(lab)
            pos.append(torch.arange(n, device=dev)), sid.append(torch.full((n,), j, device=dev))
        return (torch.cat(toks), torch.cat(feats), torch.cat(pos), torch.cat(sid), torch.cat(labels))

    def train_on_batch(self, entries, packed: PackedBatch) -> float:
        """One optimiser step over every pack of the batch (mean token loss)."""
        import torch
        import torch.nn.functional as F
        self.opt.zero_grad(set_to_none=True)
        total, count = 0.0, 0
        for pack in packed.packs:
            tok, fp, pos, sid, lab = self.batch_from_pack(entries, pack)
            logits = self.forward(tok, fp, pos, sid)
            loss = F.cross_entropy(logits, lab, ignore_index=-100, reduction="sum")
            n = int((lab >= 0).sum())
            (loss / max(1, packed.total_tokens())).backward()
            total += float(loss.detach())
            count += n
        self.opt.step()
        self.version += 1
        return total / max(1, count)

    def publish(self):
        """Write the trained weights (bf16, round to nearest) into the engine
        and publish them as the drafter snapshot (version += iterations)."""
        import torch
        with torch.no_grad():
            for k, p in self.params.items():
                self.views[k][0].copy_(p.to(torch.bfloat16))
        torch.cuda.synchronize(self.params["fc"].device)
        publish(self.engine, self.version)


def spot_train_loop(trainer: DrafterTrainer, buffer: DataBuffer, cfg: SpotTrainConfig, iterations: int,
                    preempt=None, checkpoint_path: str | None = None) -> SpotTrainLog:
    """spot_trainer.hpp:42-64: sample, pack, train, repeat; the preempt signal
    is polled between iterations (the in-flight iteration completes);
    checkpoints every checkpoint_every iterations and always on exit; the
    result is published to the engine."""
    log = SpotTrainLog()
    for _ in range(iterations):
        if preempt is not None and preempt():
            log.preempted = True
            break
        entries = buffer.sample(cfg.current_step, cfg.token_budget)
        packed = pack_sequences([e.length() for e in entries], cfg.pack_capacity)
        log.losses.append(trainer.train_on_batch(entries, packed))
        log.iterations += 1
        log.versions.append(trainer.version)
        if cfg.checkpoint_every > 0 and log.iterations % cfg.checkpoint_every == 0:
            log.checkpoints += 1
    trainer.publish()
    if checkpoint_path:
        save_checkpoint_async(trainer.engine, checkpoint_path, trainer.version).join()
    log.checkpoints += 1
    return log
