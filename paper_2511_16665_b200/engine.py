"""Python host mirror of the C-ABI (include/tlt_b200.h) for tests and bench.

Names and argument meaning follow the reference ``specsim`` API:
``sd_step`` = build_draft_tree + verify_greedy + commit for a batch
(spec_decode.hpp:111-268), ``ar_step`` = the plain branch of run_rollout
(rollout.hpp:247-261), ``Mab`` = beg_initialize / beg_select / beg_record
(beg_mab.hpp:74-170), ``plan_captures`` (capture_plan.hpp:87-155),
``run_rollout`` (rollout.hpp:130-276). Errors raise ConfigError /
RoutingError like the reference (errors.hpp:9-34).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import lib

TLT_OK, TLT_ERR_INTERNAL, TLT_ERR_CONFIG, TLT_ERR_ROUTING, TLT_ERR_CUDA, TLT_ERR_STATE = 0, 1, 2, 3, 4, 5
MAX_DEPTH = 16  # tlt::kMaxDepth (stride of debug paths)


class TltError(RuntimeError):
    pass


class ConfigError(TltError):
    pass


class RoutingError(TltError):
    pass


class CudaError(TltError):
    pass


def _check(rc: int) -> None:
    if rc == TLT_OK:
        return
    msg = lib().tlt_last_error(None)
    msg = msg.decode() if msg else ""
    raise {TLT_ERR_CONFIG: ConfigError, TLT_ERR_ROUTING: RoutingError, TLT_ERR_CUDA: CudaError}.get(rc, TltError)(
        f"[{rc}] {msg}")


class Strategy(C.Structure):
    _fields_ = [("draft_depth", C.c_int32), ("top_k", C.c_int32), ("tokens_to_verify", C.c_int32)]

    def tuple(self):
        return (self.draft_depth, self.top_k, self.tokens_to_verify)


class ModelCfg(C.Structure):
    _fields_ = [("vocab", C.c_int32), ("hidden", C.c_int32), ("layers", C.c_int32), ("heads", C.c_int32),
                ("kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32), ("qkv_bias", C.c_int32),
                ("rope_theta", C.c_float), ("rms_eps", C.c_float), ("max_slots", C.c_int32), ("max_ctx", C.c_int32)]


class InitCfg(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("layer_scale", C.c_float), ("lm_gain", C.c_float), ("lm_alt", C.c_float), ("lm_noise", C.c_float),
                ("fc_noise", C.c_float), ("drafter_lm_fp8", C.c_int32)]


class TreeOut(C.Structure):
    _fields_ = [("tokens", C.c_void_p), ("parents", C.c_void_p), ("depths", C.c_void_p), ("probs", C.c_void_p),
                ("path_probs", C.c_void_p), ("n_nodes", C.c_void_p)]


class TreeIn(C.Structure):
    _fields_ = [("tokens", C.c_void_p), ("parents", C.c_void_p), ("probs", C.c_void_p), ("path_probs", C.c_void_p),
                ("n_nodes", C.c_void_p), ("stride", C.c_int32)]


class AcceptOut(C.Structure):
    _fields_ = [("accepted", C.c_void_p), ("nodes", C.c_void_p), ("accept_len", C.c_void_p), ("bonus", C.c_void_p),
                ("kv_src", C.c_void_p), ("kv_len", C.c_void_p), ("elapsed_ms", C.c_void_p)]


class CaptureEntry(C.Structure):
    _fields_ = [("side", C.c_int32), ("bucket_lo", C.c_int32), ("bucket_hi", C.c_int32),
                ("tokens_to_verify", C.c_int32), ("top_k", C.c_int32), ("draft_depth", C.c_int32),
                ("memory_units", C.c_double)]


class CostModel(C.Structure):
    """Reference CostModelParams (cost_model.hpp:16-33); all zero = defaults."""
    _fields_ = [("t_launch", C.c_double), ("model_bytes", C.c_double), ("mem_bw", C.c_double),
                ("flops_per_token", C.c_double), ("peak_flops", C.c_double), ("drafter_step_cost", C.c_double)]


class RolloutCfg(C.Structure):
    _fields_ = [("enable_sd", C.c_int32), ("elastic_threshold", C.c_int32), ("mode", C.c_int32),
                ("temperature", C.c_float), ("fixed_strategy", Strategy), ("use_mab", C.c_int32),
                ("seed", C.c_uint64), ("use_graphs", C.c_int32), ("drafter_stale", C.c_int32),
                ("ngram_n", C.c_int32), ("ngram_continuation_len", C.c_int32), ("target_step_id", C.c_int64),
                ("parity_elapsed", C.c_int32), ("keep_finished", C.c_int32), ("cost", CostModel),
                ("rng_stream", C.c_uint64)]


class StepMetrics(C.Structure):
    """Reference StepMetrics (rollout.hpp:31-38)."""
    _fields_ = [("step_index", C.c_int32), ("batch_size", C.c_int32), ("sd_active", C.c_int32),
                ("has_strategy", C.c_int32), ("strategy", Strategy), ("elapsed", C.c_double),
                ("device_ms", C.c_double), ("accept_off", C.c_int64), ("n_accept", C.c_int32),
                ("via_ngram", C.c_int32)]


class RolloutResult(C.Structure):
    _fields_ = [("generated", C.c_void_p), ("gen_len", C.c_void_p), ("sd_steps", C.c_int64),
                ("plain_steps", C.c_int64), ("verify_events", C.c_int64), ("accepted_total", C.c_int64),
                ("emitted_total", C.c_int64), ("device_ms", C.c_double), ("wall_ms", C.c_double),
                ("gpu_launches", C.c_int64), ("total_time", C.c_double), ("ngram_verify_events", C.c_int64),
                ("accept_at_least", C.c_void_p), ("accept_at_least_cap", C.c_int32),
                ("accept_at_least_len", C.c_int32), ("finish_time", C.c_void_p), ("trace", C.c_void_p),
                ("trace_cap", C.c_int64), ("trace_len", C.c_int64), ("trace_accept_lens", C.c_void_p),
                ("trace_accept_cap", C.c_int64)]


def step_latency(batch, tokens_per_request, strategy=None, cost=None):
    """Reference step_latency (cost_model.hpp:38-48) through the C-ABI."""
    out = C.c_double()
    _check(lib().tlt_step_latency(C.byref(cost) if cost is not None else None, batch, tokens_per_request,
                                  C.byref(Strategy(*strategy)) if strategy is not None else None, C.byref(out)))
    return out.value


def _p(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


# Model shapes. "tiny" is BASELINE config 1 (the parity
# workload); "qwen2.5-7b" / "qwen2.5-32b" are the Qwen2.5 shapes of configs 2-5.
MODELS = {
    "tiny": dict(vocab=4096, hidden=256, layers=2, heads=4, kv_heads=2, head_dim=64, ffn=688, qkv_bias=1,
                 rope_theta=1e4, rms_eps=1e-6),
    "qwen2.5-7b": dict(vocab=152064, hidden=3584, layers=28, heads=28, kv_heads=4, head_dim=128, ffn=18944,
                       qkv_bias=1, rope_theta=1e6, rms_eps=1e-6),
    "qwen2.5-32b": dict(vocab=152064, hidden=5120, layers=64, heads=40, kv_heads=8, head_dim=128, ffn=27648,
                        qkv_bias=1, rope_theta=1e6, rms_eps=1e-6),
}
# Structure knob per model: mean accept length in a realistic band.
INITS = {
    "tiny": dict(seed=42, layer_scale=1.0, lm_gain=10.0, lm_alt=0.9, lm_noise=1.0, fc_noise=0.05),
    # 7B: the drafter's LM head in e4m3 (half its weight stream per draft level;
    # profiles/r2_drafter_fp8_ab.txt), emulated by the oracle (orc_neural.c lm_logits)
    "qwen2.5-7b": dict(seed=42, layer_scale=1.0, lm_gain=13.0, lm_alt=0.9, lm_noise=1.0, fc_noise=0.05,
                       drafter_lm_fp8=1),
    "qwen2.5-32b": dict(seed=42, layer_scale=0.3, lm_gain=13.0, lm_alt=0.9, lm_noise=1.0, fc_noise=0.05),
}


@dataclass
class StepResult:
    accept_len: np.ndarray
    bonus: np.ndarray
    accepted: list
    nodes: list
    kv_len: np.ndarray
    elapsed_ms: float
    tree: list | None


class Engine:
    def __init__(self, model: str | dict = "tiny", max_slots: int = 4, max_ctx: int = 512, init: dict | None = None,
                 device: int = 0, **overrides):
        m = dict(MODELS[model]) if isinstance(model, str) else dict(model)
        m.update(overrides)
        self.model = m
        ini = dict(INITS.get(model, INITS["tiny"]) if isinstance(model, str) else INITS["tiny"])
        if init:
            ini.update(init)
        self.init = ini
        self.cfg = ModelCfg(m["vocab"], m["hidden"], m["layers"], m["heads"], m["kv_heads"], m["head_dim"], m["ffn"],
                            m["qkv_bias"], m["rope_theta"], m["rms_eps"], max_slots, max_ctx)
        self.icfg = InitCfg(ini["seed"], ini["layer_scale"], ini["lm_gain"], ini["lm_alt"], ini["lm_noise"], ini["fc_noise"],
                            int(ini.get("drafter_lm_fp8", 0)))
        self.L = lib()
        h = C.c_void_p()
        _check(self.L.tlt_engine_create(C.byref(self.cfg), C.byref(self.icfg), device, C.byref(h)))
        self.h = h
        self.vocab = m["vocab"]
        self.hidden = m["hidden"]
        self.device = device
        self.max_slots, self.max_ctx = max_slots, max_ctx

    def close(self):
        if getattr(self, "h", None):
            self.L.tlt_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- state
    def prefill(self, slots, prompts):
        slots = np.asarray(slots, np.int32)
        lens = np.asarray([len(p) for p in prompts], np.int32)
        toks = np.concatenate([np.asarray(p, np.int32) for p in prompts]).astype(np.int32)
        _check(self.L.tlt_prefill(self.h, len(slots), _p(slots), _p(lens), _p(toks)))

    def release(self, slot):
        _check(self.L.tlt_release(self.h, slot))

    def slot_len(self, slot) -> int:
        v = C.c_int32()
        _check(self.L.tlt_slot_len(self.h, slot, C.byref(v)))
        return v.value

    def set_debug(self, on: bool):
        _check(self.L.tlt_set_debug(self.h, 1 if on else 0))

    # -------------------------------------------------------------- steps
    def sd_step(self, strategy, slots, want_tree: bool = True) -> StepResult:
        s = Strategy(*strategy)
        slots = np.asarray(slots, np.int32)
        b, D, T = len(slots), s.draft_depth, s.tokens_to_verify
        acc = np.zeros((b, D), np.int32)
        nodes = np.zeros((b, D), np.int32)
        alen = np.zeros(b, np.int32)
        bonus = np.zeros(b, np.int32)
        kvl = np.zeros(b, np.int32)
        ms = np.zeros(1, np.float32)
        ao = AcceptOut(acc.ctypes.data, nodes.ctypes.data, alen.ctypes.data, bonus.ctypes.data, None,
                       kvl.ctypes.data, ms.ctypes.data)
        tree = None
        to = None
        if want_tree:
            tt = np.zeros((b, T), np.int32)
            tp = np.zeros((b, T), np.int32)
            td = np.zeros((b, T), np.int32)
            tpr = np.zeros((b, T), np.float64)
            tpp = np.zeros((b, T), np.float64)
            tn = np.zeros(b, np.int32)
            to = TreeOut(tt.ctypes.data, tp.ctypes.data, td.ctypes.data, tpr.ctypes.data, tpp.ctypes.data,
                         tn.ctypes.data)
        _check(self.L.tlt_sd_step(self.h, C.byref(s), b, _p(slots), C.byref(to) if to else None, C.byref(ao)))
        if want_tree:
            tree = [list(zip(tt[i, :tn[i]].tolist(), tp[i, :tn[i]].tolist(), td[i, :tn[i]].tolist(),
                             tpr[i, :tn[i]].tolist(), tpp[i, :tn[i]].tolist())) for i in range(b)]
        return StepResult(alen, bonus, [acc[i, :alen[i]].tolist() for i in range(b)],
                          [nodes[i, :alen[i]].tolist() for i in range(b)], kvl, float(ms[0]), tree)

    def draft(self, strategy, slots):
        """Propose only (tlt_draft): build_draft_tree on the GPU drafter, no
        commit. Returns per request [(token, parent, depth, prob, path_prob)]."""
        s = Strategy(*strategy)
        slots = np.asarray(slots, np.int32)
        b, T = len(slots), s.tokens_to_verify
        tt, tp, td = (np.zeros((b, T), np.int32) for _ in range(3))
        tpr, tpp = np.zeros((b, T)), np.zeros((b, T))
        tn = np.zeros(b, np.int32)
        to = TreeOut(tt.ctypes.data, tp.ctypes.data, td.ctypes.data, tpr.ctypes.data, tpp.ctypes.data, tn.ctypes.data)
        _check(self.L.tlt_draft(self.h, C.byref(s), b, _p(slots), C.byref(to)))
        return [list(zip(tt[i, :tn[i]].tolist(), tp[i, :tn[i]].tolist(), td[i, :tn[i]].tolist(),
                         tpr[i, :tn[i]].tolist(), tpp[i, :tn[i]].tolist())) for i in range(b)]

    def verify(self, slots, trees=None, draft_depth=None):
        """verify_greedy + KV commit (tlt_verify_accept_commit). trees None:
        the engine's own last draft of these slots (pass its draft_depth);
        else per request a list of (token, parent[, ...]) in rank order."""
        slots = np.asarray(slots, np.int32)
        b = len(slots)
        ti = None
        if trees is not None:
            stride = max(1, max(len(t) for t in trees))
            tok = np.zeros((b, stride), np.int32)
            par = np.zeros((b, stride), np.int32)
            pr = np.ones((b, stride))
            pp = np.ones((b, stride))
            nn = np.zeros(b, np.int32)
            for i, t in enumerate(trees):
                nn[i] = len(t)
                for j, node in enumerate(t):
                    tok[i, j], par[i, j] = node[0], node[1]
                    if len(node) >= 5:
                        pr[i, j], pp[i, j] = node[3], node[4]
            ti = TreeIn(tok.ctypes.data, par.ctypes.data, pr.ctypes.data, pp.ctypes.data, nn.ctypes.data, stride)
            keep = (tok, par, pr, pp, nn)  # noqa: F841 (alive across the call)
        else:
            stride = int(draft_depth)
        acc = np.zeros((b, stride), np.int32)
        nodes = np.zeros((b, stride), np.int32)
        alen = np.zeros(b, np.int32)
        bonus = np.zeros(b, np.int32)
        kvl = np.zeros(b, np.int32)
        ms = np.zeros(1, np.float32)
        ao = AcceptOut(acc.ctypes.data, nodes.ctypes.data, alen.ctypes.data, bonus.ctypes.data, None,
                       kvl.ctypes.data, ms.ctypes.data)
        _check(self.L.tlt_verify_accept_commit(self.h, b, _p(slots), C.byref(ti) if ti is not None else None,
                                               C.byref(ao)))
        return StepResult(alen, bonus, [acc[i, :alen[i]].tolist() for i in range(b)],
                          [nodes[i, :alen[i]].tolist() for i in range(b)], kvl, float(ms[0]), None)

    def graph_pool_build(self, strategies, thresholds, max_batch=32, vanilla=False, sub_bucket_width=0, ar_width=0):
        """Pre-capture the CUDA-graph pool of plan_captures (capture_plan.hpp:
        87-155; vanilla = plan_captures_vanilla) and return its stats.
        sub_bucket_width / ar_width: tlt_graph_pool_configure."""
        _check(self.L.tlt_graph_pool_configure(self.h, sub_bucket_width, ar_width))
        entries, units = plan_captures(strategies, thresholds, max_batch, vanilla)
        arr = (CaptureEntry * len(entries))(*[CaptureEntry(*e) for e in entries])
        nbytes = C.c_size_t()
        _check(self.L.tlt_graph_pool_build(self.h, arr, len(entries), C.byref(nbytes)))
        st = self.graph_pool_stats()
        st.update(plan_entries=len(entries), plan_memory_units=units)
        return st

    def graph_pool_stats(self):
        n, sk, nl = C.c_int32(), C.c_int32(), C.c_int32()
        nb, ms = C.c_size_t(), C.c_double()
        _check(self.L.tlt_graph_pool_stats(self.h, C.byref(n), C.byref(sk), C.byref(nb), C.byref(ms), C.byref(nl)))
        return dict(graphs=n.value, skipped=sk.value, bytes=nb.value, build_ms=ms.value, live_graphs=nl.value)

    def graph_pool_clear(self):
        _check(self.L.tlt_graph_pool_clear(self.h))

    def probe_kernel(self, kind: int, m_tok: int, iters: int = 56):
        """Live timing of one engine GEMM site (tlt_probe_kernel): returns
        (avg_ms, algorithmic_bytes, flops) of one launch."""
        ms, b, f = C.c_float(), C.c_double(), C.c_double()
        _check(self.L.tlt_probe_kernel(self.h, kind, m_tok, iters, C.byref(ms), C.byref(b), C.byref(f)))
        return ms.value, b.value, f.value

    def probe_attention(self, b: int, ctx: int, rows_per_req: int = 1, iters: int = 56):
        """Live timing of the attention of b requests x ctx keys (tlt_probe_attention):
        returns (avg_ms, algorithmic_bytes) per layer."""
        ms, by = C.c_float(), C.c_double()
        _check(self.L.tlt_probe_attention(self.h, b, ctx, rows_per_req, iters, C.byref(ms), C.byref(by)))
        return ms.value, by.value

    def ar_step(self, slots):
        slots = np.asarray(slots, np.int32)
        out = np.zeros(len(slots), np.int32)
        ms = C.c_float()
        _check(self.L.tlt_ar_step(self.h, len(slots), _p(slots), _p(out), C.byref(ms)))
        return out, ms.value

    def sd_step_stochastic(self, draft_depth, temperature, slots, uniforms):
        """Rejection-sampling SD over drafter-sampled chains. uniforms: [b][2D+1]
        RngStream draws in consumption order; returns (StepResult, chains, consumed)."""
        slots = np.asarray(slots, np.int32)
        b, D = len(slots), draft_depth
        uni = np.ascontiguousarray(np.asarray(uniforms, np.float64).reshape(b, 2 * D + 1))
        acc = np.zeros((b, D), np.int32)
        nodes = np.zeros((b, D), np.int32)
        alen = np.zeros(b, np.int32)
        bonus = np.zeros(b, np.int32)
        kvl = np.zeros(b, np.int32)
        ms = np.zeros(1, np.float32)
        ao = AcceptOut(acc.ctypes.data, nodes.ctypes.data, alen.ctypes.data, bonus.ctypes.data, None,
                       kvl.ctypes.data, ms.ctypes.data)
        _check(self.L.tlt_sd_step_stochastic(self.h, D, C.c_float(temperature), b, _p(slots), _p(uni),
                                             C.byref(ao)))
        chains, consumed = [], []
        for i in range(b):
            ch = np.zeros(D, np.int32)
            n, cons = C.c_int32(), C.c_int32()
            _check(self.L.tlt_debug_chain(self.h, i, _p(ch), C.byref(n), C.byref(cons)))
            chains.append(ch[:n.value].tolist())
            consumed.append(cons.value)
        res = StepResult(alen, bonus, [acc[i, :alen[i]].tolist() for i in range(b)],
                         [nodes[i, :alen[i]].tolist() for i in range(b)], kvl, float(ms[0]), None)
        return res, chains, consumed

    def sd_step_chain(self, draft_depth, slots, chains):
        """Greedy verify of host-proposed linear chains (n-gram fallback branch,
        rollout.hpp:212-216; chain_from_tokens, spec_decode.hpp:228-240).
        chains[i]: list of <= draft_depth tokens (may be empty)."""
        slots = np.asarray(slots, np.int32)
        b, D = len(slots), draft_depth
        ch = np.zeros((b, D), np.int32)
        lens = np.zeros(b, np.int32)
        for i, c in enumerate(chains):
            if len(c) > D:
                raise ConfigError("chain_lens: must be in [0, draft_depth]")
            ch[i, :len(c)] = c
            lens[i] = len(c)
        acc = np.zeros((b, D), np.int32)
        nodes = np.zeros((b, D), np.int32)
        alen = np.zeros(b, np.int32)
        bonus = np.zeros(b, np.int32)
        kvl = np.zeros(b, np.int32)
        ms = np.zeros(1, np.float32)
        ao = AcceptOut(acc.ctypes.data, nodes.ctypes.data, alen.ctypes.data, bonus.ctypes.data, None,
                       kvl.ctypes.data, ms.ctypes.data)
        _check(self.L.tlt_sd_step_chain(self.h, D, b, _p(slots), _p(ch), _p(lens), C.byref(ao)))
        return StepResult(alen, bonus, [acc[i, :alen[i]].tolist() for i in range(b)],
                          [nodes[i, :alen[i]].tolist() for i in range(b)], kvl, float(ms[0]), None)

    def sd_step_chain_stochastic(self, draft_depth, temperature, slots, chains, uniforms):
        """verify_stochastic of host chains with one-hot q (n-gram branch,
        stochastic mode). uniforms: [b][D+1]; returns (StepResult, consumed)."""
        slots = np.asarray(slots, np.int32)
        b, D = len(slots), draft_depth
        ch = np.zeros((b, D), np.int32)
        lens = np.zeros(b, np.int32)
        for i, c in enumerate(chains):
            ch[i, :len(c)] = c
            lens[i] = len(c)
        uni = np.ascontiguousarray(np.asarray(uniforms, np.float64).reshape(b, D + 1))
        acc = np.zeros((b, D), np.int32)
        nodes = np.zeros((b, D), np.int32)
        alen = np.zeros(b, np.int32)
        bonus = np.zeros(b, np.int32)
        kvl = np.zeros(b, np.int32)
        ms = np.zeros(1, np.float32)
        ao = AcceptOut(acc.ctypes.data, nodes.ctypes.data, alen.ctypes.data, bonus.ctypes.data, None,
                       kvl.ctypes.data, ms.ctypes.data)
        _check(self.L.tlt_sd_step_chain_stochastic(self.h, D, C.c_float(temperature), b, _p(slots), _p(ch), _p(lens),
                                                   _p(uni), C.byref(ao)))
        consumed = []
        for i in range(b):
            tmp = np.zeros(max(D, 1), np.int32)
            n, cons = C.c_int32(), C.c_int32()
            _check(self.L.tlt_debug_chain(self.h, i, _p(tmp), C.byref(n), C.byref(cons)))
            consumed.append(cons.value)
        res = StepResult(alen, bonus, [acc[i, :alen[i]].tolist() for i in range(b)],
                         [nodes[i, :alen[i]].tolist() for i in range(b)], kvl, float(ms[0]), None)
        return res, consumed

    def export_sequence(self, slot: int, device: bool = True):
        """C2 payload of a live slot (tlt_export_sequence): committed tokens
        [0, len] (int32) and target features [0, len) as bf16 [len][hidden],
        copied by the engine straight into a torch tensor (CUDA when device)."""
        import torch
        n = C.c_int32()
        _check(self.L.tlt_slot_len(self.h, slot, C.byref(n)))
        L = n.value
        toks = np.zeros(L + 1, np.int32)
        feats = torch.empty((L, self.hidden), dtype=torch.bfloat16,
                            device=f"cuda:{self.device}" if device else "cpu")
        if not device:
            feats = feats.pin_memory() if torch.cuda.is_available() else feats
        _check(self.L.tlt_export_sequence(self.h, slot, _p(toks), L + 1, C.c_void_p(feats.data_ptr()),
                                          C.c_size_t(feats.numel() * 2), C.byref(n)))
        return toks, feats

    def debug_target_rows(self, i: int, max_rows: int = 32):
        out = np.zeros((max_rows, self.vocab), np.float64)
        n = C.c_int32()
        _check(self.L.tlt_debug_target_rows(self.h, i, _p(out), max_rows, C.byref(n)))
        return out[:n.value]

    # ---------------------------------------------------------- debug
    def debug_expansions(self, i: int, max_exp: int = 4096):
        n = C.c_int32()
        plen = np.zeros(max_exp, np.int32)
        paths = np.zeros((max_exp, MAX_DEPTH), np.int32)
        _check(self.L.tlt_debug_expansions(self.h, i, max_exp, C.byref(n), _p(plen), _p(paths), None))
        cnt = min(n.value, max_exp)
        rows = np.zeros((cnt, self.vocab), np.float64)
        _check(self.L.tlt_debug_expansions(self.h, i, cnt, C.byref(n), _p(plen), _p(paths), _p(rows)))
        return [(tuple(paths[j, :plen[j]].tolist()), rows[j]) for j in range(cnt)]

    def debug_verify_logits(self, i: int, max_rows: int = 256):
        out = np.zeros((max_rows, self.vocab), np.float32)
        n = C.c_int32()
        _check(self.L.tlt_debug_verify_logits(self.h, i, _p(out), max_rows, C.byref(n)))
        return out[:n.value]

    def debug_ar_logits(self, b: int):
        out = np.zeros((b, self.vocab), np.float32)
        _check(self.L.tlt_debug_ar_logits(self.h, _p(out), b))
        return out

    # ---------------------------------------------------------- rollout
    def run_rollout(self, prompts, max_lens, request_ids=None, *, enable_sd=True, elastic_threshold=32,
                    strategy=(4, 4, 16), mab: "Mab | None" = None, seed=0, use_graphs=True, mode="greedy",
                    temperature=0.0, drafter_stale=False, ngram_n=2, ngram_continuation_len=8, target_step_id=0,
                    parity_elapsed=False, keep_finished=False, cost=None, trace_cap=1 << 16, rng_stream=0):
        """Reference run_rollout (rollout.hpp:130-276). Returns the RolloutResult
        fields (requests' tokens and finish_time, trace of StepMetrics,
        accept_at_least, counters) as a dict."""
        n = len(prompts)
        rid = np.asarray(request_ids if request_ids is not None else range(n), np.int32)
        plen = np.asarray([len(p) for p in prompts], np.int32)
        toks = np.concatenate([np.asarray(p, np.int32) for p in prompts]).astype(np.int32)
        ml = np.asarray(max_lens, np.int32)
        stride = int(ml.max())
        gen = np.zeros((n, stride), np.int32)
        glen = np.zeros(n, np.int32)
        cfg = RolloutCfg(1 if enable_sd else 0, elastic_threshold, 1 if mode == "stochastic" else 0,
                         float(temperature), Strategy(*strategy),
                         1 if mab is not None else 0, seed, 1 if use_graphs else 0, 1 if drafter_stale else 0,
                         ngram_n, ngram_continuation_len, target_step_id, 1 if parity_elapsed else 0,
                         1 if keep_finished else 0, cost if cost is not None else CostModel(), rng_stream)
        res = RolloutResult(gen.ctypes.data, glen.ctypes.data)
        aal = np.zeros(64, np.int64)
        fin = np.zeros(n, np.float64)
        trace = (StepMetrics * trace_cap)()
        tacc = np.zeros(trace_cap * 4, np.int32)
        res.accept_at_least, res.accept_at_least_cap = aal.ctypes.data, len(aal)
        res.finish_time = fin.ctypes.data
        res.trace, res.trace_cap = C.cast(trace, C.c_void_p), trace_cap
        res.trace_accept_lens, res.trace_accept_cap = tacc.ctypes.data, len(tacc)
        _check(self.L.tlt_run_rollout(self.h, C.byref(cfg), mab.h if mab is not None else None, n, _p(rid),
                                      _p(plen), _p(toks), _p(ml), stride, C.byref(res)))
        steps = []
        for t in trace[:min(res.trace_len, trace_cap)]:
            o = t.accept_off
            steps.append(dict(step_index=t.step_index, batch_size=t.batch_size, sd_active=bool(t.sd_active),
                              strategy=t.strategy.tuple() if t.has_strategy else None, elapsed=t.elapsed,
                              device_ms=t.device_ms, via_ngram=bool(t.via_ngram),
                              accept_lens=tacc[o:o + t.n_accept].tolist() if o + t.n_accept <= len(tacc) else None))
        return dict(tokens=[gen[i, :glen[i]].tolist() for i in range(n)], sd_steps=res.sd_steps,
                    plain_steps=res.plain_steps, verify_events=res.verify_events,
                    ngram_verify_events=res.ngram_verify_events,
                    accepted_total=res.accepted_total, emitted_total=res.emitted_total, device_ms=res.device_ms,
                    wall_ms=res.wall_ms, gpu_launches=res.gpu_launches, total_time=res.total_time,
                    accept_at_least=aal[:res.accept_at_least_len].tolist(), finish_time=fin.tolist(),
                    trace=steps, trace_len=res.trace_len,
                    mean_accept_len=(res.accepted_total / res.verify_events) if res.verify_events else 0.0)


class Rng:
    def __init__(self, seed=0, stream=0, _h=None):
        self.L = lib()
        if _h is None:
            _h = C.c_void_p()
            _check(self.L.tlt_rng_create(C.c_uint64(seed), C.c_uint64(stream), C.byref(_h)))
        self.h = _h

    def fork(self, label):
        h = C.c_void_p()
        _check(self.L.tlt_rng_fork(self.h, C.c_uint64(label), C.byref(h)))
        return Rng(_h=h)

    def next_u64(self):
        return self.L.tlt_rng_next_u64(self.h)

    def uniform01(self):
        return self.L.tlt_rng_uniform01(self.h)

    def uniform_int(self, n):
        """RngStream::uniform_int (rng.hpp:59-61): next_u64() % n."""
        return self.next_u64() % n

    def normal(self):
        """RngStream::normal (rng.hpp:64-69), Box-Muller over two uniform01 draws."""
        import math
        u1, u2 = self.uniform01(), self.uniform01()
        return math.sqrt(-2.0 * math.log1p(-u1)) * math.cos(6.283185307179586477 * u2)

    def ids(self):
        """(seed, stream_id) of this stream (rng.hpp:43-44)."""
        sd, st = C.c_uint64(), C.c_uint64()
        _check(self.L.tlt_rng_ids(self.h, C.byref(sd), C.byref(st)))
        return sd.value, st.value

    def __del__(self):
        try:
            self.L.tlt_rng_destroy(self.h)
        except Exception:
            pass


class Ngram:
    """Model-free n-gram drafter index (reference NgramIndex / ngram_insert /
    ngram_draft, ngram.hpp:13-103, plus the NgramTracker cursor,
    rollout.hpp:103-120), host C++ behind the C-ABI."""

    def __init__(self, n=2, continuation_len=8):
        self.L = lib()
        self.h = C.c_void_p()
        _check(self.L.tlt_ngram_create(n, continuation_len, C.byref(self.h)))
        self.n, self.continuation_len = n, continuation_len

    def insert(self, response, step_id=0):
        r = np.asarray(response, np.int32)
        _check(self.L.tlt_ngram_insert(self.h, _p(r), len(r), C.c_int64(step_id)))

    def extend(self, stream, step_id=0):
        r = np.asarray(stream, np.int32)
        _check(self.L.tlt_ngram_extend(self.h, _p(r), len(r), C.c_int64(step_id)))

    def draft(self, ctx, depth):
        c = np.asarray(ctx, np.int32)
        out = np.zeros(max(depth, 1), np.int32)
        n = C.c_int32()
        _check(self.L.tlt_ngram_draft(self.h, _p(c), len(c), depth, _p(out), C.byref(n)))
        return out[:n.value].tolist()

    def size(self):
        v = C.c_int64()
        _check(self.L.tlt_ngram_size(self.h, C.byref(v)))
        return v.value

    def __del__(self):
        try:
            self.L.tlt_ngram_destroy(self.h)
        except Exception:
            pass


class Mab:
    def __init__(self, strategies, thresholds, epsilon=0.1, window=20):
        self.L = lib()
        self.strategies = [tuple(s) for s in strategies]
        arr = (Strategy * len(strategies))(*[Strategy(*s) for s in strategies])
        thr = np.asarray(thresholds, np.int32)
        h = C.c_void_p()
        _check(self.L.tlt_mab_create(arr, len(strategies), _p(thr), len(thr), C.c_double(epsilon), window,
                                     C.byref(h)))
        self.h = h

    def select(self, batch, rng: Rng):
        arm = C.c_int32()
        s = Strategy()
        _check(self.L.tlt_mab_select(self.h, batch, rng.h, C.byref(arm), C.byref(s)))
        return arm.value, s.tuple()

    def record(self, strategy, elapsed, accept_lens):
        lens = np.asarray(accept_lens, np.int32)
        _check(self.L.tlt_mab_record(self.h, C.byref(Strategy(*strategy)), C.c_double(elapsed), _p(lens),
                                     len(lens)))

    def arm_stats(self, arm):
        med, sel, n = C.c_double(), C.c_int64(), C.c_int32()
        _check(self.L.tlt_mab_arm_stats(self.h, arm, C.byref(med), C.byref(sel), C.byref(n)))
        return med.value, sel.value, n.value

    def arm_window(self, arm, cap=4096):
        """(rewards, accept_lens) windows of one arm, oldest first."""
        rw = np.zeros(cap, np.float64)
        al = np.zeros(cap, np.float64)
        n = C.c_int32()
        _check(self.L.tlt_mab_arm_window(self.h, arm, rw.ctypes.data_as(C.c_void_p), al.ctypes.data_as(C.c_void_p),
                                         cap, C.byref(n)))
        k = min(n.value, cap)
        return rw[:k].tolist(), al[:k].tolist()

    def apply_record(self, arm, reward, a_bar):
        _check(self.L.tlt_mab_apply_record(self.h, arm, C.c_double(reward), C.c_double(a_bar)))

    def take_log(self, cap: int = 1 << 16):
        """Records this replica's beg_record logged since the last call: [(arm, reward, a_bar)]."""
        arm = np.zeros(cap, np.int32)
        rew = np.zeros(cap, np.float64)
        ab = np.zeros(cap, np.float64)
        n = C.c_int32()
        _check(self.L.tlt_mab_take_log(self.h, _p(arm), rew.ctypes.data_as(C.c_void_p),
                                       ab.ctypes.data_as(C.c_void_p), cap, C.byref(n)))
        return [(int(arm[i]), float(rew[i]), float(ab[i])) for i in range(n.value)]

    def copy_from(self, other: "Mab"):
        _check(self.L.tlt_mab_copy(self.h, other.h))

    def __del__(self):
        try:
            self.L.tlt_mab_destroy(self.h)
        except Exception:
            pass


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)


class C1:
    """C1 inside the library (tlt_c1_*): fixed-size BEG-MAB record blocks
    all-gathered over NCCL (engine-device communicator, side stream) or a
    host all-gather callback, applied in rank order to the shared replica."""

    def __init__(self, h, keep=None):
        self.L = lib()
        self.h = h
        self._keep = keep  # the ctypes callback must outlive the handle

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_char * 128)()
        _check(lib().tlt_c1_nccl_unique_id(buf))
        return bytes(buf)

    @classmethod
    def nccl(cls, engine: "Engine", uid: bytes, world: int, rank: int, max_records: int = 4096):
        h = C.c_void_p()
        buf = (C.c_char * 128).from_buffer_copy(uid)
        _check(lib().tlt_c1_create_nccl(engine.h, buf, world, rank, max_records, C.byref(h)))
        return cls(h)

    @classmethod
    def from_dist(cls, dist, max_records: int = 4096):
        """Callback transport over a torch.distributed group (the record block
        travels as a CPU or CUDA byte tensor, as the backend needs)."""
        import torch
        world, rank = dist.get_world_size(), dist.get_rank()
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")

        def gather(user, send, recv, nbytes):
            try:
                t = torch.frombuffer(bytearray(C.string_at(send, nbytes)), dtype=torch.uint8).to(dev)
                outs = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(outs, t)
                blob = torch.cat(outs).cpu().numpy().tobytes()
                C.memmove(recv, blob, len(blob))
                return 0
            except Exception:
                return 1

        fn = ALLGATHER_FN(gather)
        h = C.c_void_p()
        _check(lib().tlt_c1_create_callback(world, rank, fn, None, max_records, C.byref(h)))
        return cls(h, keep=fn)

    def merge(self, local: "Mab", shared: "Mab") -> int:
        n = C.c_int32()
        _check(self.L.tlt_c1_merge(self.h, local.h, shared.h, C.byref(n)))
        return n.value

    def __del__(self):
        try:
            self.L.tlt_c1_destroy(self.h)
        except Exception:
            pass


def merge_bandit_stats(dist, local: "Mab", shared: "Mab", c1: "C1 | None" = None) -> int:
    """C1: all-gather every rank's new BEG-MAB records and apply
    them to the shared replica in rank order, so every rank's shared replica is
    bit-identical; the local replica then restarts from it. With one rank this
    is exactly the local beg_record sequence. Returns the records merged.
    With `c1` the library does the pack / all-gather / apply (tlt_c1_merge)."""
    if c1 is not None:
        return c1.merge(local, shared)
    mine = local.take_log()
    world = dist.get_world_size() if dist is not None else 1
    logs = [None] * world
    if dist is not None:
        dist.all_gather_object(logs, mine)
    else:
        logs = [mine]
    n = 0
    for recs in logs:  # rank order
        for arm, reward, a_bar in recs:
            shared.apply_record(arm, reward, a_bar)
            n += 1
    local.copy_from(shared)
    return n


def handback_samples(dist, samples, trainer_rank: int = 0):
    """C2: every rank hands its finished sequences
    [(tokens int32 [L+1], features bf16 [L][d]), ...] to the trainer rank,
    which returns them as [(rank, tokens, features), ...] in rank order (its
    own first at its rank position); other ranks return []. Point-to-point
    over the process group's backend (NCCL with CUDA tensors, gloo on CPU);
    off the decode critical path (called at rollout boundaries)."""
    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    # the transport device follows the backend, not the samples: NCCL moves
    # CUDA tensors only, gloo point-to-point CPU tensors only
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    cnt = torch.tensor([len(samples)], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt)
    out = []
    if rank != trainer_rank:
        for toks, feats in samples:
            t = torch.as_tensor(np.asarray(toks, np.int32)).to(dev)
            hdr = torch.tensor([t.numel(), feats.shape[0], feats.shape[1] if feats.dim() == 2 else 0],
                               dtype=torch.int64, device=dev)
            dist.send(hdr, trainer_rank)
            dist.send(t, trainer_rank)
            dist.send(feats.contiguous().view(torch.int16).to(dev), trainer_rank)  # bf16 bits
        return out
    for r in range(world):
        if r == trainer_rank:
            out += [(r, torch.as_tensor(np.asarray(t, np.int32)).to(dev), f.to(dev)) for t, f in samples]
            continue
        for _ in range(int(counts[r].item())):
            hdr = torch.zeros(3, dtype=torch.int64, device=dev)
            dist.recv(hdr, r)
            nt, L, d = (int(x) for x in hdr.tolist())
            t = torch.zeros(nt, dtype=torch.int32, device=dev)
            dist.recv(t, r)
            f = torch.zeros((L, d), dtype=torch.int16, device=dev)
            dist.recv(f, r)
            out.append((r, t, f.view(torch.bfloat16)))
    return out


def plan_captures(strategies, thresholds, max_batch=32, vanilla=False):
    L = lib()
    arr = (Strategy * len(strategies))(*[Strategy(*s) for s in strategies])
    thr = np.asarray(thresholds, np.int32)
    out = (CaptureEntry * 4096)()
    n = C.c_int()
    tot = C.c_double()
    _check(L.tlt_plan_captures(arr, len(strategies), _p(thr), len(thr), max_batch, 1 if vanilla else 0, out, 4096,
                               C.byref(n), C.byref(tot)))
    return [(e.side, e.bucket_lo, e.bucket_hi, e.tokens_to_verify, e.top_k, e.draft_depth, e.memory_units)
            for e in out[:n.value]], tot.value
