"""bench.py — accepted tokens/s of the greedy tree-SD rollout (BASELINE config 2).

One bench STEP = one rollout of the rank's request group (Qwen2.5-7B-shaped
random-init target + 1-layer EAGLE drafter; 64 requests per GPU, long-tail
response lengths, batch 64 -> 1) through the reference-facing C-ABI
(tlt_run_rollout == reference run_rollout, rollout.hpp:130-276): prefill,
elastic gate (SD when batch < 32), BEG-MAB strategy select per batch bucket
(default 8 arms, thresholds {1,2,8,16}), greedy tree SD steps replaying the
CUDA-graph pool, plain AR steps above the gate, emission with EOS / max_len.

  value  = emitted tokens (all ranks) / device time of the timed rollouts
           (CUDA events on the engine stream around every prefill/step, max
           over ranks) — inputs already resident.
  e2e    = same tokens / wall time of the timed tlt_run_rollout calls with
           HOST prompts in and HOST generated tokens out (all H2D/D2H and
           per-step host decisions inside), barrier + synchronize on both
           sides, max over ranks.

Under torchrun each rank runs an independent engine on its own GPU with its
own 64 requests (request_id % world == rank, weak scaling); no collective is
on the data path. --impl reference times the CPU path (oracle port of the
reference spec_generate over the neural leaves) on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "accepted tokens/s per GPU (tree-SD rollout) at 1/2/4/8 B200; mean accept len"
DEFAULT_ARMS = [(10, 8, 64), (6, 8, 64), (10, 8, 48), (6, 8, 48), (10, 8, 32), (6, 8, 32), (10, 8, 16), (6, 8, 16)]
THRESHOLDS = [1, 2, 8, 16]


def peaks():
    """(HBM GB/s, dense bf16 TFLOP/s burst, sustained, source): the driver-measured
    MEASURED_PEAKS.json, else the B200_PROFILING.md fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return (float(p["hbm_gbs"]), float(p["bf16_tflops"]),
                float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), "measured")
    except Exception:
        return 6650.0, 1590.0, 1373.0, "fallback"


def model_costs(m, drafter_fp8=False):
    """Algorithmic bytes / flops of the Qwen-shaped target and the EAGLE drafter
    (SURVEY.md 8(d)): weights streamed per forward (the embedding is a row
    gather), KV bytes per token, matmul flops per row. drafter_fp8: the
    drafter's LM head streams one byte per weight (+ a scale per row) and its
    flops run at twice the bf16 rate (counted as half as many bf16 flops)."""
    d, L, H, KV, hd, F, V = (m[k] for k in ("hidden", "layers", "heads", "kv_heads", "head_dim", "ffn", "vocab"))
    nqkv = (H + 2 * KV) * hd
    mat_layer = d * nqkv + H * hd * d + 2 * d * F + F * d
    layer_b = (mat_layer + nqkv + 2 * d) * 2
    lm_d = V * d + V * 4 if drafter_fp8 else V * d * 2
    return dict(
        target_w=L * layer_b + V * d * 2 + d * 2,
        drafter_w=(2 * d * d) * 2 + layer_b + lm_d + d * 2,
        kv_tok=L * 2 * KV * hd * 2, dkv_tok=2 * KV * hd * 2,
        fl_row_t=2 * (L * mat_layer + V * d),
        fl_row_d=2 * (2 * d * d + mat_layer) + (V * d if drafter_fp8 else 2 * V * d),
        attn_fl=4 * H * hd, layers=L)


def step_roofline(m, b, ctx, strategy, bw_gbs, tflops, drafter_fp8=False):
    """t_roof of one engine step = sum over phases of max(bytes / BW, flops /
    peak). strategy None = plain AR decode (R = b rows);
    else (D, k, T): D drafter levels (level 1: b LM rows, level l: b *
    min(T, k^(l-1)) rows) + one verify forward over b (T + 1) rows."""
    c = model_costs(m, drafter_fp8)
    bw, pk = bw_gbs * 1e9, tflops * 1e12

    def phase(w, rows, kv_read, kv_write, attn_rows_keys, fl_row, layers):
        byts = w + kv_read + kv_write
        fl = rows * fl_row + c["attn_fl"] * layers * attn_rows_keys
        return max(byts / bw, fl / pk), byts, fl

    if strategy is None:
        t, byts, fl = phase(c["target_w"], b, b * ctx * c["kv_tok"], b * c["kv_tok"], b * (ctx + 1), c["fl_row_t"],
                            c["layers"])
        return dict(t_roof_ms=t * 1e3, bytes=byts, flops=fl)
    D, k, T = strategy
    tot_t, tot_b, tot_f = 0.0, 0.0, 0.0
    for lv in range(1, D + 1):
        rows = b if lv == 1 else b * min(T, k ** (lv - 1))
        t, byts, fl = phase(c["drafter_w"], rows, b * ctx * c["dkv_tok"], rows * c["dkv_tok"], rows * (ctx + lv), c["fl_row_d"], 1)
        tot_t, tot_b, tot_f = tot_t + t, tot_b + byts, tot_f + fl
    R = b * (T + 1)
    t, byts, fl = phase(c["target_w"], R, b * ctx * c["kv_tok"], R * c["kv_tok"], R * (ctx + (T + 1) / 2),
                        c["fl_row_t"], c["layers"])
    return dict(t_roof_ms=(tot_t + t) * 1e3, bytes=tot_b + byts, flops=tot_f + fl)


def response_lengths(n, mu, sigma, max_len, seed):
    """sample_response_length (rollout.hpp:42-50) with the RngStream normal (rng.hpp:64-69)."""
    from paper_2511_16665_b200.engine import Rng
    r = Rng(seed, 0x4C454E)
    out = []
    for _ in range(n):
        u1, u2 = r.uniform01(), r.uniform01()
        z = math.sqrt(-2.0 * math.log1p(-u1)) * math.cos(6.283185307179586477 * u2)
        v = round(math.exp(mu + sigma * z))
        out.append(int(min(max(v, 1), max_len)))
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, device):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                o = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                    "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                f = [x.strip() for x in o.stdout.strip().split(",")]
                if len(f) >= 7:
                    self.samples.append(f)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    return world, rank, local, pg


def max_over_ranks(pg, vals, local):
    if pg is None:
        return vals
    import torch
    t = torch.tensor(vals, dtype=torch.float64, device=f"cuda:{local}")
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return t.tolist()


def sum_over_ranks(pg, vals, local):
    if pg is None:
        return vals
    import torch
    t = torch.tensor(vals, dtype=torch.float64, device=f"cuda:{local}")
    pg.all_reduce(t, op=pg.ReduceOp.SUM)
    return t.tolist()


def barrier(pg, local):
    import torch
    torch.cuda.synchronize(local)
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize(local)


# ----------------------------------------------------------------- CPU arm
def cpu_rollout_sample(model_name, n_threads, gen_tokens, prompt_len, strategy, seed=0):
    """Oracle port of spec_generate (greedy tree) over the neural CPU leaves."""
    import ctypes as C

    import oracle as O
    from paper_2511_16665_b200.engine import INITS, MODELS
    m, ini = MODELS[model_name], INITS[model_name]
    L = O.orc()
    cfg = O.ModelCfg(m["vocab"], m["hidden"], m["layers"], m["heads"], m["kv_heads"], m["head_dim"], m["ffn"],
                     m["qkv_bias"], m["rope_theta"], m["rms_eps"], prompt_len + gen_tokens + 64)
    icfg = O.InitCfg(ini["seed"], ini["layer_scale"], ini["lm_gain"], ini["lm_alt"], ini["lm_noise"],
                     ini["fc_noise"], int(ini.get("drafter_lm_fp8", 0)))
    t0 = time.time()
    om = L.orc_model_create(C.byref(cfg), C.byref(icfg), n_threads)
    init_s = time.time() - t0
    L.orc_neural_spec_generate.argtypes = [C.c_void_p] * 11
    rng = np.random.default_rng(seed)
    prompt = (C.c_int32 * prompt_len)(*rng.integers(2, m["vocab"], prompt_len).tolist())
    out = (C.c_int32 * 512)()
    n = C.c_int()
    acc = (C.c_int32 * 512)()
    t0 = time.time()
    steps = L.orc_neural_spec_generate(om, prompt, prompt_len, gen_tokens, C.byref(O.Strategy(*strategy)), out,
                                       C.byref(n), acc, None, None, 512)
    dt = time.time() - t0
    L.orc_model_destroy(om)
    return dict(tokens=n.value, seconds=dt, steps=steps, init_s=init_s,
                mean_accept=float(np.mean(list(acc[:max(steps, 1)]))))


def cpu_rows(model_name, prompt_len, strategy):
    """CPU baseline: the oracle port of the reference hot path
    (C restatement of spec_generate over the neural CPU leaves) on this host.
    b = 1 with 1 thread and with all cores; b in {8, 32} with all cores, each
    request run to one SD step (max_len 2) as the reference's per-request loop
    does (rollout.hpp:191 is sequential over requests)."""
    import ctypes as C

    import oracle as O
    from paper_2511_16665_b200.engine import INITS, MODELS
    m, ini = MODELS[model_name], INITS[model_name]
    L = O.orc()
    cfg = O.ModelCfg(m["vocab"], m["hidden"], m["layers"], m["heads"], m["kv_heads"], m["head_dim"], m["ffn"],
                     m["qkv_bias"], m["rope_theta"], m["rms_eps"], prompt_len + 64)
    icfg = O.InitCfg(ini["seed"], ini["layer_scale"], ini["lm_gain"], ini["lm_alt"], ini["lm_noise"],
                     ini["fc_noise"], int(ini.get("drafter_lm_fp8", 0)))
    cores = os.cpu_count() or 1
    om = L.orc_model_create(C.byref(cfg), C.byref(icfg), cores)
    L.orc_neural_spec_generate.argtypes = [C.c_void_p] * 11
    L.orc_model_set_threads.argtypes = [C.c_void_p, C.c_int]
    rng = np.random.default_rng(0)

    def run(b, threads):
        L.orc_model_set_threads(om, threads)
        toks, t0 = 0, time.time()
        for _ in range(b):
            prompt = (C.c_int32 * prompt_len)(*rng.integers(2, m["vocab"], prompt_len).tolist())
            out = (C.c_int32 * 64)()
            n = C.c_int()
            acc = (C.c_int32 * 64)()
            L.orc_neural_spec_generate(om, prompt, prompt_len, 2, C.byref(O.Strategy(*strategy)), out, C.byref(n),
                                       acc, None, None, 64)
            toks += n.value
        dt = time.time() - t0
        return {"b": b, "threads": threads, "tokens": toks, "seconds": round(dt, 2),
                "tokens_per_s": round(toks / dt, 4)}

    rows = [run(1, 1), run(1, cores), run(8, cores), run(32, cores)]
    L.orc_model_destroy(om)
    return rows, cores


def lscpu_model():
    try:
        o = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in o.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(a):
    world, rank, local, pg = dist_setup(a.gpus)
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    strategy = (6, 8, 16)
    vals = []
    for i in range(a.warmup + a.steps):
        r = cpu_rollout_sample(a.model, threads, a.cpu_gen, a.cpu_prompt, strategy, seed=i)
        if i >= a.warmup:
            vals.append(r)
    toks = sum(v["tokens"] for v in vals)
    secs = sum(v["seconds"] for v in vals)
    value = toks / secs if secs > 0 else 0.0
    sample = (f"{a.model} CPU oracle port, 1 request, prompt {a.cpu_prompt}, {a.cpu_gen} generated tokens per step, "
              f"greedy tree SD {strategy}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "tokens/s", "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(secs / max(1, len(vals)) * 1e3, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16-weights/fp32",
        "data": "synthetic", "config": {"workload": "config2-long-tail-sample", "model": a.model},
        "cpu_baseline": {"value": round(value, 4), "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "mean_accept_len": round(float(np.mean([v["mean_accept"] for v in vals])), 3)}), flush=True)


# ----------------------------------------------------------------- GPU arm
PROBES = [  # (name, probe kind, M, bound)  -- SURVEY.md 8(d) per-kernel rooflines
    ("gate_up GEMM+SwiGLU, long-tail verify (b=1, T=16)", 0, 17, "hbm"),
    ("gate_up GEMM+SwiGLU, plain decode b=1", 0, 1, "hbm"),
    ("down GEMM+residual, long-tail verify (b=1, T=16)", 2, 17, "hbm"),
    ("LM head + fused top-1, long-tail verify (b=1, T=16)", 4, 17, "hbm"),
    ("gate_up GEMM+SwiGLU, verify b=31 T=16", 0, 527, "tensor"),
    ("down GEMM+residual, verify b=31 T=16", 2, 527, "tensor"),
    ("LM head bf16 -> fp32 logits, 496 rows (drafter level width at b=31)", 3, 496, "tensor"),
    ("drafter LM head as configured (7B: e4m3) -> fp32 logits, drafter level b=1 (8 rows)", 6, 8, "hbm"),
    ("gate_up GEMM+SwiGLU, verify b=16 T=64", 0, 1040, "tensor"),
]


ATTN_PROBES = [  # (name, requests, committed keys, query rows per request)
    ("attention (flash-decode + combine), plain decode b=64 ctx=1024", 64, 1024, 1),
    ("attention (flash-decode + combine), plain decode b=1 ctx=1024", 1, 1024, 1),
    ("tree attention (+combine), verify b=5 T=48 ctx=700", 5, 700, 49),
    ("tree attention (+combine), verify b=31 T=16 ctx=700", 31, 700, 17),
]


def traffic_table():
    """dram bytes per launch from the committed ncu captures: round 1's --set
    full GEMM captures, overridden by round 2's per-site engine probes
    (tools/traffic_json.py over tools/gpu_r2_s3_final.sh)."""
    out = {}
    for name in ("r1_traffic.json", "r2_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                out.update({k: v for k, v in json.load(f).items() if not k.startswith("_")})
        except Exception:
            pass
    return out


def kernel_rooflines(eng, peak_gbs, peak_tf, peak_kind):
    """Each probe: the engine's own GEMM site, successive layers' weights,
    CUDA events on the engine stream (tlt_probe_kernel; best of 5 timed
    passes of 56 launches after a warm-up pass)."""
    traffic = traffic_table()
    out = []
    for name, kind, m, bound in PROBES:
        print(f"[bench] probe {name}", file=sys.stderr, flush=True)
        ms, byts, flops = eng.probe_kernel(kind, m, 56)
        if bound == "hbm":
            ach = byts / (ms * 1e-3) / 1e9
            rec = {"kernel": name, "bound": "hbm", "achieved": round(ach, 1), "peak": peak_gbs, "unit": "GB/s",
                   "frac": round(ach / peak_gbs, 3)}
        else:
            ach = flops / (ms * 1e-3) / 1e12
            rec = {"kernel": name, "bound": "tensor", "achieved": round(ach, 1), "peak": peak_tf, "unit": "TFLOP/s",
                   "frac": round(ach / peak_tf, 3)}
        t = traffic.get(f"{kind}:{m}")
        rec.update({"traffic": t, "algorithmic_bytes": int(byts), "M": m, "avg_launch_ms": round(ms, 4),
                    "peak_kind": peak_kind})
        out.append(rec)
    for name, bb, ctx, rpr in ATTN_PROBES:
        print(f"[bench] probe {name}", file=sys.stderr, flush=True)
        ms, byts = eng.probe_attention(bb, ctx, rpr, 56)
        ach = byts / (ms * 1e-3) / 1e9
        out.append({"kernel": name, "bound": "hbm", "achieved": round(ach, 1), "peak": peak_gbs, "unit": "GB/s",
                    "frac": round(ach / peak_gbs, 3), "traffic": None, "algorithmic_bytes": int(byts),
                    "M": bb * rpr, "avg_launch_ms": round(ms, 4), "peak_kind": peak_kind})
    return out


# Per-bucket fixed-step rows (the 2x bar is about b < 32): the reference
# default arms of each BEG-MAB bucket (T = 64 / 48 / 32 / 16 for buckets
# [1,1] / [2,7] / [8,15] / [16,32], experiment.hpp:87-95, beg_mab.hpp:95-105).
BUCKET_ROWS = [(1, [(10, 8, 64), (6, 8, 64)]), (4, [(10, 8, 48), (6, 8, 48)]), (8, [(10, 8, 32), (6, 8, 32)]),
               (16, [(10, 8, 16), (6, 8, 16)]), (31, [(10, 8, 16), (6, 8, 16)])]


def bucket_rows(eng, a, peak_gbs, peak_tf_sus):
    """b requests: prefill (prompt a.prompt), `warm_ar` untimed plain steps
    (generated context), then `steps` timed AR steps and, per default arm, 2
    warm SD steps (drafter catch-up + graph capture) and `steps` timed SD
    steps. Tokens/s are device time (CUDA events per step); the step
    roofline is t_roof / t_measured."""
    rows = []
    V = eng.vocab
    steps, warm_ar = a.bucket_steps, a.bucket_ctx
    for b, arms in BUCKET_ROWS:
        rng = np.random.default_rng(77 + b)
        prompts = [rng.integers(2, V, a.prompt).tolist() for _ in range(b)]
        slots = list(range(b))
        for s in slots:
            eng.release(s)
        eng.prefill(slots, prompts)
        for _ in range(warm_ar):
            eng.ar_step(slots)
        ctx = a.prompt - 1 + warm_ar
        ar_ms = 0.0
        for _ in range(steps):
            ar_ms += eng.ar_step(slots)[1]
        ctx += steps
        ar_tps = b * steps / (ar_ms / 1e3)
        ar_roof = step_roofline(eng.model, b, ctx, None, peak_gbs, peak_tf_sus)["t_roof_ms"]
        row = {"b": b, "ctx": ctx, "ar_tok_s": round(ar_tps, 1), "ar_ms_per_step": round(ar_ms / steps, 3),
               "ar_step_roofline_frac": round(ar_roof / (ar_ms / steps), 3), "arms": []}
        for arm in arms:
            for _ in range(2):
                eng.sd_step(arm, slots, want_tree=False)
            ms, emitted, acc = 0.0, 0, 0
            L0 = [eng.slot_len(s) for s in slots]
            for _ in range(steps):
                r = eng.sd_step(arm, slots, want_tree=False)
                ms += r.elapsed_ms
                emitted += int(r.accept_len.sum()) + b
                acc += int(r.accept_len.sum())
            ctx_sd = int(np.mean(L0))
            roof = step_roofline(eng.model, b, ctx_sd, arm, peak_gbs, peak_tf_sus,
                                 bool(eng.init.get("drafter_lm_fp8", 0)))["t_roof_ms"]
            tps = emitted / (ms / 1e3)
            row["arms"].append({"strategy": list(arm), "sd_tok_s": round(tps, 1), "speedup_vs_ar": round(tps / ar_tps, 3),
                                "ms_per_step": round(ms / steps, 3), "mean_accept_len": round(acc / (b * steps), 3),
                                "step_roofline_frac": round(roof / (ms / steps), 3), "ctx": ctx_sd})
        row["best_speedup_vs_ar"] = max(x["speedup_vs_ar"] for x in row["arms"])
        rows.append(row)
        print(f"[bench] bucket b={b}: {row}", file=sys.stderr, flush=True)
    return rows


GEMM_SITES = [(1, "qkv (+bias, RoPE, KV write)"), (5, "o-proj (+residual)"), (0, "gate_up (+SwiGLU)"),
              (2, "down (+residual)")]


def gemm_class(eng, M, bound, peak_gbs, peak_tf):
    """The dominant kernel class over one target forward at M rows: every
    tcgen05 GEMM site of a layer (each timed over successive layers' weights,
    tlt_probe_kernel, CUDA events on the engine stream) x layers + the LM
    head with the fused top-1 epilogue. achieved = summed algorithmic bytes
    (or flops) / summed launch time."""
    L = eng.model["layers"]
    t = byts = fl = 0.0
    parts = []
    tt = traffic_table()
    traffic = 0.0
    for kind, name in GEMM_SITES:
        ms, b_, f_ = eng.probe_kernel(kind, M, 56)
        t, byts, fl = t + ms * L, byts + b_ * L, fl + f_ * L
        tr = tt.get(f"{kind}:{M}")
        traffic = traffic + tr * L if (tr is not None and traffic is not None) else None
        parts.append({"site": name, "avg_launch_us": round(ms * 1e3, 2), "bytes": int(b_), "flops": int(f_),
                      "traffic": tr})
    ms, b_, f_ = eng.probe_kernel(4, M, 8)
    t, byts, fl = t + ms, byts + b_, fl + f_
    tr = tt.get(f"4:{M}")
    traffic = traffic + tr if (tr is not None and traffic is not None) else None
    parts.append({"site": "LM head (+fused top-1)", "avg_launch_us": round(ms * 1e3, 2), "bytes": int(b_),
                  "flops": int(f_), "traffic": tr})
    traffic = int(traffic) if traffic is not None else None  # ncu DRAM bytes of one forward's GEMMs
    if bound == "hbm":
        ach = byts / (t * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": round(ach, 1), "peak": peak_gbs, "unit": "GB/s",
                "frac": round(ach / peak_gbs, 3), "traffic": traffic, "M": M, "forward_gemm_ms": round(t, 3),
                "algorithmic_bytes": int(byts), "sites": parts}
    ach = fl / (t * 1e-3) / 1e12
    return {"bound": "tensor", "achieved": round(ach, 1), "peak": peak_tf, "unit": "TFLOP/s",
            "frac": round(ach / peak_tf, 3), "traffic": traffic, "M": M, "forward_gemm_ms": round(t, 3),
            "flops": int(fl), "sites": parts}


def token_match(sd_tokens, ar_tokens):
    """Greedy SD is lossless vs plain decode (spec_decode.hpp:349-350): compare
    the SD rollout's tokens with the AR rollout's on the same workload."""
    same, tot, first_div, identical = 0, 0, [], 0
    for s, r in zip(sd_tokens, ar_tokens):
        n = min(len(s), len(r))
        k = next((j for j in range(n) if s[j] != r[j]), n)
        same += k
        tot += max(len(s), len(r))
        identical += int(s == r)
        if s != r:
            first_div.append(k)
    return {"requests": len(sd_tokens), "identical_requests": identical,
            "prefix_match_rate": round(same / max(1, tot), 6), "first_divergence_positions": first_div[:16]}


def divergence_margins(eng, prompts, sd_tokens, ar_tokens, limit=16, atol=0.05, rtol=0.01):
    """At each diverging request's first SD/AR difference: the target's fp32
    logits for the two candidate tokens, from a prefill of prompt ++ the
    common prefix and one debug plain-decode step. Greedy SD is lossless up to
    floating-point near-ties of the top-2 target logits (the verify forward
    runs another row batch / GEMM tiling than plain decode, so bf16 rounding
    differs); a margin within the tests' tolerance (tests/parity_util.py
    greedy_streams_agree: 2 (atol + rtol |logit|)) is a tie, not an error."""
    out = []
    eng.set_debug(True)
    try:
        for p, s, r in zip(prompts, sd_tokens, ar_tokens):
            if s == r or len(out) >= limit:
                continue
            k = next((j for j in range(min(len(s), len(r))) if s[j] != r[j]), None)
            if k is None:  # one stream is a prefix of the other (EOS / max_len cut)
                continue
            eng.prefill([0], [p + r[:k]])
            eng.ar_step([0])
            lg = eng.debug_ar_logits(1)[0]
            eng.release(0)
            a, b = float(lg[r[k]]), float(lg[s[k]])
            top2 = np.sort(lg)[-2:]
            out.append({"pos": k, "margin": abs(a - b), "tol": 2 * (atol + rtol * max(abs(a), abs(b))),
                        "top2_gap": float(top2[1] - top2[0])})
    finally:
        eng.set_debug(False)
    return {"checked": len(out), "within_tol": sum(1 for x in out if x["margin"] <= x["tol"]),
            "max_margin": round(max((x["margin"] for x in out), default=0.0), 5),
            "min_tol": round(min((x["tol"] for x in out), default=0.0), 5),
            "note": "first SD/AR divergences: |logit(ar tok) - logit(sd tok)| of the target at that position vs "
                    "2 (0.05 + 0.01 |logit|); within tol = a floating-point near-tie"}


def run_ours(a):
    world, rank, local, pg = dist_setup(a.gpus)
    import torch
    torch.cuda.set_device(local)
    from paper_2511_16665_b200.engine import Engine, Mab, merge_bandit_stats
    peak_gbs, peak_tf, peak_tf_sus, peak_kind = peaks()
    n = a.requests
    max_ctx = a.prompt + a.max_len + 8
    eng = Engine(a.model, max_slots=n, max_ctx=max_ctx, device=local)
    # the CUDA-graph pool of plan_captures (capture_plan.hpp:87-126), pre-built
    # before the timed region: one fused step graph per (bucket, strategy),
    # replayed for every batch of its bucket; padded plain-decode sizes
    pool = (eng.graph_pool_build(DEFAULT_ARMS, THRESHOLDS, 32, sub_bucket_width=a.pool_sub_width,
                                 ar_width=a.pool_ar_width) if a.graph_pool else None)
    if pool is not None:
        pool.update(sub_bucket_width=a.pool_sub_width, ar_width=a.pool_ar_width)
    mab = Mab(DEFAULT_ARMS, THRESHOLDS, 0.1, 20)
    # C1: with several ranks each rank's bandit records are all-gathered after
    # every rollout and merged in rank order into a shared replica (NCCL; the
    # only collective besides the timing reductions)
    mab_shared = Mab(DEFAULT_ARMS, THRESHOLDS, 0.1, 20) if pg is not None else None
    c1 = None
    if pg is not None:  # C1 inside the library: NCCL communicator on the engine's device, side stream
        from paper_2511_16665_b200.engine import C1
        uid = [C1.nccl_unique_id() if rank == 0 else None]
        pg.broadcast_object_list(uid, src=0)
        c1 = C1.nccl(eng, uid[0], world, rank)
    V = eng.vocab

    def workload(step):
        # request ids of this rank: global id = rank + world * i (request_id % world == rank)
        ids = [rank + world * i for i in range(n)]
        rng = np.random.default_rng(1000 * step + rank)
        prompts = [rng.integers(2, V, a.prompt).tolist() for _ in range(n)]
        lens = response_lengths(n, math.log(a.len_median), a.len_sigma, a.max_len, seed=100 + step + 7919 * rank)
        return ids, prompts, lens

    buf = None
    if a.spot_train_iters > 0:  # TLT spot training: the warmup rollouts feed the drafter's trainer (untimed)
        from paper_2511_16665_b200 import spot as S
        buf = S.DataBuffer(retention=1)

    def rollout(step, enable_sd=True, collect=False):
        ids, prompts, lens = workload(step)
        r = eng.run_rollout(prompts, lens, ids, enable_sd=enable_sd, elastic_threshold=a.elastic,
                            mab=mab, seed=step, use_graphs=True, keep_finished=collect)
        if collect:  # C2: every finished sequence (tokens + target features) into the DataBuffer
            toks, feats = [], []
            for i in range(n):
                t, f = eng.export_sequence(i)
                toks.append(t.tolist())
                feats.append(f)
                eng.release(i)
            buf.insert(step, toks, feats)
        if mab_shared is not None and enable_sd:
            r["c1_records"] = merge_bandit_stats(pg, mab, mab_shared, c1)
        return r

    spot = None
    for s in range(a.warmup):
        r = rollout(s, collect=buf is not None)
        print(f"[bench] warmup rollout {s} done", file=sys.stderr, flush=True)
    if buf is not None:
        t0 = time.perf_counter()
        tr = S.DrafterTrainer(eng, lr=a.spot_lr)
        cfg = S.SpotTrainConfig(current_step=a.warmup - 1, token_budget=a.spot_budget, pack_capacity=2048)
        lg = S.spot_train_loop(tr, buf, cfg, a.spot_train_iters)
        spot = {"iterations": lg.iterations, "drafter_version": S.drafter_version(eng),
                "loss_first": round(lg.losses[0], 4), "loss_last": round(lg.losses[-1], 4),
                "buffer_sequences": len(buf.entries), "train_s": round(time.perf_counter() - t0, 1),
                "note": "EAGLE drafter spot-trained on the warmup rollouts' own sequences (C2 export), untimed, "
                        "before the timed rollouts (TLT's adaptive drafter)"}
        del buf, tr
        import torch
        torch.cuda.empty_cache()
        print(f"[bench] spot training {spot}", file=sys.stderr, flush=True)
    barrier(pg, local)
    res = []
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for s in range(a.steps):
            res.append(rollout(a.warmup + s))
        barrier(pg, local)
        wall = time.perf_counter() - t0
    # where the rollout time goes (trace of the timed rollouts): device ms and
    # emitted tokens per batch range, SD vs plain steps
    def time_split(rs):
        bins = [("ar_b>=32", lambda m: not m["sd_active"]), ("sd_b16-31", lambda m: m["sd_active"] and m["batch_size"] >= 16),
                ("sd_b8-15", lambda m: m["sd_active"] and 8 <= m["batch_size"] < 16),
                ("sd_b2-7", lambda m: m["sd_active"] and 2 <= m["batch_size"] < 8),
                ("sd_b1", lambda m: m["sd_active"] and m["batch_size"] == 1)]
        tot = sum(m["device_ms"] for r in rs for m in r["trace"])
        out = {}
        for name, f in bins:
            ms = sum(m["device_ms"] for r in rs for m in r["trace"] if f(m))
            steps = sum(1 for r in rs for m in r["trace"] if f(m))
            toks = sum((sum(m["accept_lens"]) + m["batch_size"]) if m["sd_active"] else m["batch_size"]
                       for r in rs for m in r["trace"] if f(m))
            out[name] = {"time_frac": round(ms / tot, 4) if tot else 0.0, "steps": steps,
                         "tokens_per_s": round(toks / (ms / 1e3), 1) if ms else None}
        return out
    split = time_split(res)
    emitted = sum(r["emitted_total"] for r in res)
    dev_s = sum(r["device_ms"] for r in res) / 1e3
    accepted = sum(r["accepted_total"] for r in res)
    events = sum(r["verify_events"] for r in res)
    launches = sum(r["gpu_launches"] for r in res)
    sd_steps = sum(r["sd_steps"] for r in res)
    plain_steps = sum(r["plain_steps"] for r in res)
    h2d = sum(4 * (a.prompt + 3) * n for _ in range(1))
    d2h = 4 * sum(len(t) for t in res[-1]["tokens"]) if res else 0
    tot = sum_over_ranks(pg, [emitted, accepted, events], local)
    mx = max_over_ranks(pg, [dev_s, wall], local)
    value = tot[0] / mx[0] if mx[0] > 0 else 0.0
    e2e = tot[0] / mx[1] if mx[1] > 0 else 0.0
    # same engine, plain AR decode on the same workload (the 2x denominator)
    ar = rollout(a.warmup, enable_sd=False) if a.ar_baseline else None
    ar_tok_s = ar["emitted_total"] / (ar["device_ms"] / 1e3) if ar else None
    sd_same = res[0] if res else None
    match = token_match(sd_same["tokens"], ar["tokens"]) if (ar and sd_same) else None
    if match is not None and rank == 0 and match["identical_requests"] < match["requests"]:
        match["divergences"] = divergence_margins(eng, workload(a.warmup)[1], sd_same["tokens"], ar["tokens"])
    out = None
    if rank == 0:
        print("[bench] probes", file=sys.stderr, flush=True)
        kernels = kernel_rooflines(eng, peak_gbs, peak_tf, peak_kind)
        roof = gemm_class(eng, 17, "hbm", peak_gbs, peak_tf)
        roof["kernel"] = ("tcgen05 GEMM class, one long-tail verify forward (b=1, T=16: M=17): qkv+o+gate_up+down "
                          "x layers + LM head/top-1")
        roof_tc = gemm_class(eng, 527, "tensor", peak_gbs, peak_tf)
        roof_tc["kernel"] = "tcgen05 GEMM class, one verify forward at b=31, T=16 (M=527)"
        buckets = bucket_rows(eng, a, peak_gbs, peak_tf_sus) if a.bucket_steps > 0 else None
        cpu = None
        if a.cpu_rows:
            rows_c, cores = cpu_rows(a.model, a.cpu_prompt, (6, 8, 16))
            allc = [r for r in rows_c if r["threads"] == cores]
            tps = sum(r["tokens"] for r in allc) / sum(r["seconds"] for r in allc)
            cpu = {"value": round(tps, 4), "unit": "tokens/s", "cores": cores, "kind": "port",
                   "cpu_model": lscpu_model(), "rows": rows_c,
                   "sample": f"{a.model} CPU oracle port (C restatement of spec_generate over the neural leaves), "
                             f"prompt {a.cpu_prompt}, greedy tree SD (6,8,16), each request to its first SD step "
                             f"(max_len 2); rows b=1 at 1 thread and all cores, b=8 and b=32 at all cores; value = "
                             f"all-core tokens / all-core seconds"}
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": "tokens/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(mx[0] * 1e3 / max(1, a.steps), 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "config2: Qwen2.5-7B-shaped random-init target + 1-layer EAGLE drafter, "
                                   "long-tail rollout batch 64->1, greedy tree SD, BEG-MAB",
                       "model": a.model, "requests_per_gpu": n, "prompt_len": a.prompt,
                       "len_lognormal": [round(math.log(a.len_median), 4), a.len_sigma, a.max_len],
                       "elastic_threshold": a.elastic, "strategies": DEFAULT_ARMS, "thresholds": THRESHOLDS,
                       "parallelism": f"dp{world} (independent rollout groups)",
                       "l2": "KV + weights (15.2 GB) exceed the 126 MB L2 every step; no flush needed"},
            "per_gpu": round(value / world, 2),
            "mean_accept_len": round(tot[1] / tot[2], 3) if tot[2] else None,
            "mean_accept_len_with_bonus": round(tot[1] / tot[2] + 1, 3) if tot[2] else None,
            "sd_steps": sd_steps, "plain_steps": plain_steps,
            "e2e": {"value": round(e2e, 2), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "graph_pool": pool,
            "spot_training": spot,
            "time_split": split,
            "roofline": roof,
            "roofline_tensor_class": roof_tc,
            "per_bucket": buckets,
            "kernels": kernels,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        if ar is not None:
            out["ar_baseline"] = {"value": round(ar_tok_s, 2), "unit": "tokens/s (same engine, plain AR decode)",
                                  "sd_rollout_same_workload": round(sd_same["emitted_total"] /
                                                                    (sd_same["device_ms"] / 1e3), 2),
                                  "speedup": round((sd_same["emitted_total"] / (sd_same["device_ms"] / 1e3)) /
                                                   ar_tok_s, 3),
                                  "token_match_sd_vs_ar": match}
        print(json.dumps(out), flush=True)
    eng.close()
    if pg is not None:
        pg.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--requests", type=int, default=64)
    ap.add_argument("--prompt", type=int, default=256)
    # response lengths lognormal(mu = ln 1500, sigma 1), max 8192
    ap.add_argument("--len-median", type=float, default=1500.0)
    ap.add_argument("--len-sigma", type=float, default=1.0)
    ap.add_argument("--max-len", type=int, default=8192)
    ap.add_argument("--graph-pool", type=int, default=1)
    ap.add_argument("--spot-train-iters", type=int, default=0)
    ap.add_argument("--spot-lr", type=float, default=3e-5)
    ap.add_argument("--spot-budget", type=int, default=65536)
    # 0: one graph per plan bucket (padding to the bucket's largest batch);
    # w: sub-buckets of <= w batch sizes (DESIGN.md §6 measures the trade-off)
    ap.add_argument("--pool-sub-width", type=int, default=1)
    ap.add_argument("--pool-ar-width", type=int, default=1)
    ap.add_argument("--elastic", type=int, default=32)
    ap.add_argument("--ar-baseline", type=int, default=1)
    ap.add_argument("--cpu-gen", type=int, default=8)
    ap.add_argument("--cpu-prompt", type=int, default=8)
    ap.add_argument("--cpu-rows", type=int, default=1)
    ap.add_argument("--bucket-steps", type=int, default=12)
    ap.add_argument("--bucket-ctx", type=int, default=400, help="untimed plain steps before the bucket rows")
    a = ap.parse_args()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
