"""run_experiment / emit_report on the GPU engine.

Reference: experiment.hpp — ExperimentConfig (:27-100) with its JSON schema
(unknown keys rejected with the field path, :104-124, 235-371),
run_experiment (:435-695) and emit_report (:741-832). Per RL step the
long-tail workload is drawn from the experiment's RngStream (prompt tokens
uniform in [2, V), response budgets from sample_response_length, forks 100+s
/ 200+s), rolled out once WITHOUT speculative decoding (the baseline arm,
rng fork 300+s) and once with the adaptive engine (elastic gate, BEG-MAB
over the strategies, rng fork 400+s) on the same requests, and the per-step
table, acceptance-by-position curve, bandit state, capture-plan comparison
and speedup curve are reported in the reference's JSON / CSV formats.

What changes on the GPU: time is the measured device time of each engine
step (CUDA events, ms) instead of the cost model's units, unless
``parity_elapsed`` replays the reference's step_latency clock; the target is
the random-init neural model (no Markov drift between RL steps); the
capture comparison adds the REAL device bytes of the bucketed and vanilla
CUDA-graph pools next to the plan's memory units; the speedup curve is
measured (one fixed-strategy SD step vs one plain step per (batch, T)) next
to the reference's analytic sd_speedup. Spot drafter training (the idle-
worker trainer, coordinator, checkpoints: SURVEY.md §8 f3) is not part of
this harness: drafter_version stays 0, training_iterations 0, match_rate
is not measured (reported as 0) and coord_events is empty.
"""
from __future__ import annotations

import copy
import json
import math
import os

import numpy as np

from .engine import INITS, MODELS, ConfigError, CostModel, Engine, Mab, Rng, plan_captures, step_latency

DEFAULT_STRATEGIES = [(d, 8, v) for v in (64, 48, 32, 16) for d in (10, 6)]  # experiment.hpp:87-95

DEFAULTS = {
    "seed": 42,
    "rl_steps": 4,
    "model": "tiny",
    "elastic_threshold": 32,
    "mode": "greedy_tree",
    "temperature": 0.0,
    "parity_elapsed": False,
    "use_graph_pool": True,
    "ngram": {"n": 2, "continuation_len": 8},
    "drafter": {"staleness_bound": 1, "stale": False},
    "strategies": [list(s) for s in DEFAULT_STRATEGIES],
    "mab": {"epsilon": 0.1, "window": 20, "thresholds": [1, 2, 8, 16], "max_capture_batch": 32},
    "cost": {"t_launch": 0.05, "model_bytes": 1.0, "mem_bw": 1.0, "flops_per_token": 1.0, "peak_flops": 377.0,
             "drafter_step_cost": 0.046},
    "calibration_emitted": {"16": 4.45, "32": 4.85, "48": 5.05, "64": 5.18},
    "workload": {"mu": 5.2, "sigma": 1.0, "max_len": 1024, "requests_per_step": 64, "prompt_len": 2},
    "speedup_curve": {"batches": [1, 2, 4, 8, 16, 32], "ctx": 256},
}


def _check_keys(j, path, allowed):
    """experiment.hpp:104-114: objects only, unknown keys rejected by field path."""
    if not isinstance(j, dict):
        raise ConfigError(f"[2] {path or '<root>'}: must be an object")
    for k in j:
        if k not in allowed:
            raise ConfigError(f"[2] {(path + '.' + k) if path else k}: unknown key")


def config_from_json(j: dict) -> dict:
    """Merge a JSON document over the defaults (reference config_from_json)."""
    _check_keys(j, "", DEFAULTS.keys())
    cfg = copy.deepcopy(DEFAULTS)
    for k, v in j.items():
        if isinstance(DEFAULTS[k], dict) and k not in ("calibration_emitted",):
            _check_keys(v, k, DEFAULTS[k].keys())
            cfg[k].update(v)
        else:
            cfg[k] = v
    validate(cfg)
    return cfg


def validate(c: dict) -> None:
    """ExperimentConfig::validate (experiment.hpp:128-160) for the fields used here."""
    def bad(field, msg):
        raise ConfigError(f"[2] {field}: {msg}")
    if c["rl_steps"] < 1:
        bad("rl_steps", "must be >= 1")
    if c["elastic_threshold"] < 1:
        bad("elastic_threshold", "must be >= 1")
    if c["mode"] not in ("greedy_tree", "stochastic_linear"):
        bad("mode", "must be greedy_tree or stochastic_linear")
    if c["mode"] == "stochastic_linear" and not c["temperature"] > 0:
        bad("target.temperature", "stochastic_linear requires temperature > 0")  # :136-137
    if c["model"] not in MODELS:
        bad("model", "unknown model shape")
    w = c["workload"]
    if w["requests_per_step"] < 1:
        bad("workload.requests_per_step", "must be >= 1")
    if w["max_len"] < 1:
        bad("workload.max_len", "must be >= 1")
    if w["sigma"] < 0:
        bad("workload.sigma", "must be >= 0")
    if w["prompt_len"] < 1:
        bad("workload.prompt_len", "must be >= 1")
    if not c["strategies"]:
        bad("strategies", "must not be empty")
    for f, v in c["cost"].items():
        if not v > 0:
            bad(f"cost_model.{f}", "must be > 0")


def sample_response_length(mu, sigma, max_len, rng: Rng) -> int:
    """rollout.hpp:42-50 (truncated log-normal, mass beyond max_len on max_len)."""
    raw = math.exp(mu + sigma * rng.normal())
    r = math.floor(raw)  # std::round: half away from zero (raw > 0)
    if raw - r >= 0.5:
        r += 1
    if r < 1:
        return 1
    return int(min(r, max_len))


def _percentile(values, q):
    """experiment.hpp:417-424."""
    if not values:
        return 0
    v = sorted(values)
    rank = max(1, math.ceil(q * len(v)))
    return v[min(rank - 1, len(v) - 1)]


def _cost(c):
    k = c["cost"]
    return CostModel(k["t_launch"], k["model_bytes"], k["mem_bw"], k["flops_per_token"], k["peak_flops"],
                     k["drafter_step_cost"])


def _analytic_speedup(c, batch, s):
    """sd_speedup (cost_model.hpp:83-88) with the configured calibration profile."""
    cal = {int(k): v for k, v in c["calibration_emitted"].items()}
    T = s[2]
    if T in cal:
        em = cal[T]
    else:
        ks = sorted(cal)
        if T <= ks[0]:
            em = cal[ks[0]]
        elif T >= ks[-1]:
            em = cal[ks[-1]]
        else:
            hi = next(k for k in ks if k > T)
            lo = max(k for k in ks if k < T)
            em = cal[lo] + (T - lo) / (hi - lo) * (cal[hi] - cal[lo])
    base = step_latency(batch, 1, None, _cost(c))
    sd = step_latency(batch, T, s, _cost(c))
    return em * base / sd


def run_experiment(cfg: dict | None = None, engine: Engine | None = None, max_ctx: int | None = None,
                   keep_tokens: bool = False) -> dict:
    """experiment.hpp:435-695 on the GPU engine; returns the RunReport as the
    reference's report_to_json document (plus GPU-only fields; keep_tokens
    adds both arms' token streams per step under "_tokens")."""
    c = config_from_json(cfg or {})
    strategies = [tuple(s) for s in c["strategies"]]
    w = c["workload"]
    root = Rng(c["seed"], 0)
    V = MODELS[c["model"]]["vocab"]
    n = w["requests_per_step"]
    own = engine is None
    if own:
        engine = Engine(c["model"], max_slots=max(n, c["mab"]["max_capture_batch"]),
                        max_ctx=max_ctx or (w["prompt_len"] + w["max_len"] + 160))
    mab_cfg = c["mab"]
    thr = mab_cfg["thresholds"]
    cap_batch = max(mab_cfg["max_capture_batch"], thr[-1])
    report = {"config": c, "steps": []}
    # capture comparison: plan units (reference) + the real pools on this GPU
    rep = {}
    for s in strategies:
        rep.setdefault(s[2], s)
    rep_list = [rep[t] for t in sorted(rep, reverse=True)]
    bucketed, units_b = plan_captures(rep_list, thr, cap_batch)
    vanilla, units_v = plan_captures(rep_list, thr, cap_batch, vanilla=True)

    def plan_json(entries, total):
        return {"entries": [{"side": "TARGET" if e[0] == 0 else "DRAFT", "bucket_lo": e[1], "bucket_hi": e[2],
                             "tokens_to_verify": e[3], "top_k": e[4], "draft_depth": e[5], "memory_units": e[6]}
                            for e in entries], "total_memory_units": total}

    cc = {"bucketed": plan_json(bucketed, units_b), "vanilla": plan_json(vanilla, units_v), "ratio": units_v / units_b}
    gv = engine.graph_pool_build(strategies, thr, cap_batch, vanilla=True)
    gb = engine.graph_pool_build(strategies, thr, cap_batch)
    cc["device_bytes"] = {"bucketed": gb["bytes"], "vanilla": gv["bytes"],
                          "bucketed_graphs": gb["graphs"], "vanilla_graphs": gv["graphs"],
                          "bucketed_build_ms": gb["build_ms"], "vanilla_build_ms": gv["build_ms"]}
    if not c["use_graph_pool"]:
        engine.graph_pool_clear()
    mab = Mab(strategies, thr, mab_cfg["epsilon"], mab_cfg["window"])
    mode = "stochastic" if c["mode"] == "stochastic_linear" else "greedy"
    common = dict(elastic_threshold=c["elastic_threshold"], mode=mode, temperature=c["temperature"],
                  drafter_stale=c["drafter"]["stale"], ngram_n=c["ngram"]["n"],
                  ngram_continuation_len=c["ngram"]["continuation_len"], parity_elapsed=c["parity_elapsed"],
                  cost=_cost(c), use_graphs=True)
    tot_base = tot_tlt = 0.0
    at_least, tot_events = [], 0
    for step in range(c["rl_steps"]):
        len_rng = root.fork(100 + step)
        prompt_rng = root.fork(200 + step)
        prompts, max_lens = [], []
        for _ in range(n):
            prompts.append([2 + prompt_rng.uniform_int(V - 2) for _ in range(w["prompt_len"])])
            max_lens.append(sample_response_length(w["mu"], w["sigma"], w["max_len"], len_rng))
        base_rng = root.fork(300 + step)
        tlt_rng = root.fork(400 + step)
        base = engine.run_rollout(prompts, max_lens, enable_sd=False, seed=base_rng.ids()[0],
                                  rng_stream=base_rng.ids()[1], **common)
        tlt = engine.run_rollout(prompts, max_lens, enable_sd=True, mab=mab, seed=tlt_rng.ids()[0],
                                 rng_stream=tlt_rng.ids()[1], **common)
        lens = [len(t) for t in base["tokens"]]
        sr = {"step": step, "baseline_time": base["total_time"], "tlt_time": tlt["total_time"],
              "speedup": base["total_time"] / tlt["total_time"], "mean_len": sum(lens) / len(lens),
              "p50_len": _percentile(lens, 0.5), "p75_len": _percentile(lens, 0.75), "max_len": max(lens),
              "mean_accept": tlt["mean_accept_len"], "sd_steps": tlt["sd_steps"], "plain_steps": tlt["plain_steps"],
              "verify_events": tlt["verify_events"], "ngram_verify_events": tlt["ngram_verify_events"],
              "drafter_version": 0, "match_rate": 0.0, "snapshot_published": False, "training_iterations": 0,
              "coord_events": {}, "mab_selections": [mab.arm_stats(i)[1] for i in range(len(strategies))],
              # GPU-only: emitted tokens and tokens/s of both arms, greedy losslessness
              "baseline_tokens_per_s": sum(lens) / (base["device_ms"] / 1e3),
              "tlt_tokens_per_s": tlt["emitted_total"] / (tlt["device_ms"] / 1e3),
              "tokens_match": (tlt["tokens"] == base["tokens"]) if mode == "greedy" else None,
              "tokens_first_divergence": [next((j for j in range(min(len(a), len(b_))) if a[j] != b_[j]),
                                               min(len(a), len(b_))) if a != b_ else -1
                                          for a, b_ in zip(tlt["tokens"], base["tokens"])]}
        if len(at_least) < len(tlt["accept_at_least"]):
            at_least += [0] * (len(tlt["accept_at_least"]) - len(at_least))
        for i, v in enumerate(tlt["accept_at_least"]):
            at_least[i] += v
        tot_events += tlt["verify_events"]
        tot_base += base["total_time"]
        tot_tlt += tlt["total_time"]
        report["steps"].append(sr)
        if keep_tokens:
            report.setdefault("_tokens", []).append({"prompts": prompts, "tlt": tlt["tokens"],
                                                     "baseline": base["tokens"]})
    report["aggregate_speedup"] = tot_base / tot_tlt
    report["accept_rate_by_position"] = [v / tot_events if tot_events else 0.0 for v in at_least]
    groups = {}
    for i, s in enumerate(strategies):
        groups.setdefault(s[2], []).append(i)
    report["mab_state"] = {
        "epsilon": mab_cfg["epsilon"], "window": mab_cfg["window"], "thresholds": thr,
        "groups": [groups[t] for t in sorted(groups, reverse=True)],
        "arms": [{"strategy": {"draft_depth": s[0], "top_k": s[1], "tokens_to_verify": s[2]},
                  "rewards": mab.arm_window(i)[0], "accept_lens": mab.arm_window(i)[1],
                  "selections": mab.arm_stats(i)[1]} for i, s in enumerate(strategies)]}
    report["capture_comparison"] = cc
    # speedup curve: analytic (reference) + measured on this engine
    curve = []
    sc = c["speedup_curve"]
    for batch in sc["batches"]:
        for T in sorted(rep):
            s = rep[T]
            pt = {"batch": batch, "tokens_to_verify": T, "speedup": _analytic_speedup(c, batch, s)}
            if batch <= engine.max_slots:
                pt["measured"] = _measured_speedup(engine, batch, s, sc["ctx"], V)
            curve.append(pt)
    report["speedup_curve"] = curve
    report["model"] = {"name": c["model"], **MODELS[c["model"]], "init": INITS[c["model"]]}
    if own:
        engine.close()
    return report


def _measured_speedup(engine: Engine, batch, s, ctx, V):
    """Emitted tokens per device-ms of fixed-strategy SD steps over plain
    steps at this batch (prefilled ctx-token prompts, 3 steps each)."""
    rng = np.random.default_rng(batch * 1000 + s[2])
    slots = list(range(batch))
    prompts = [rng.integers(2, V, ctx).tolist() for _ in slots]
    engine.prefill(slots, prompts)
    ar_ms = 0.0
    for _ in range(3):
        _, ms = engine.ar_step(slots)
        ar_ms += ms
    sd_ms, emitted = 0.0, 0
    for _ in range(3):
        r = engine.sd_step(s, slots, want_tree=False)
        sd_ms += r.elapsed_ms
        emitted += int(r.accept_len.sum()) + batch
    for sl in slots:
        engine.release(sl)
    return (emitted / sd_ms) / (3 * batch / ar_ms)


def _fmt(v):
    """experiment.hpp:426-430 fmt_double: %.12g."""
    return "%.12g" % v


def emit_report(report: dict, fmt: str, out_dir: str) -> list:
    """experiment.hpp:741-832: json -> report.json; csv -> steps.csv,
    accept_position.csv, speedup_vs_batch.csv, capture_memory.csv,
    reward_trace.csv (same columns and number format). Byte-stable for
    identical reports."""
    if fmt not in ("csv", "json"):
        raise ConfigError("[2] format: must be csv or json")
    try:
        os.makedirs(out_dir, exist_ok=True)
    except OSError:
        raise ConfigError(f"[2] out: cannot create output directory: {out_dir}")
    if fmt == "json":
        with open(os.path.join(out_dir, "report.json"), "w") as f:
            f.write(json.dumps(report, indent=2) + "\n")
        return ["report.json"]
    written = []

    def w(name, lines):
        with open(os.path.join(out_dir, name), "w", newline="") as f:
            f.write("".join(l + "\n" for l in lines))
        written.append(name)

    w("steps.csv", ["step,baseline_time,tlt_time,speedup,mean_len,p50_len,p75_len,max_len,mean_accept,sd_steps,"
                    "plain_steps,verify_events,ngram_verify_events,drafter_version,match_rate,training_iterations"] +
      [",".join([str(s["step"]), _fmt(s["baseline_time"]), _fmt(s["tlt_time"]), _fmt(s["speedup"]),
                 _fmt(s["mean_len"]), str(s["p50_len"]), str(s["p75_len"]), str(s["max_len"]),
                 _fmt(s["mean_accept"]), str(s["sd_steps"]), str(s["plain_steps"]), str(s["verify_events"]),
                 str(s["ngram_verify_events"]), str(s["drafter_version"]), _fmt(s["match_rate"]),
                 str(s["training_iterations"])]) for s in report["steps"]])
    w("accept_position.csv", ["position,accept_rate"] +
      [f"{i + 1},{_fmt(v)}" for i, v in enumerate(report["accept_rate_by_position"])])
    w("speedup_vs_batch.csv", ["batch,tokens_to_verify,speedup"] +
      [f"{p['batch']},{p['tokens_to_verify']},{_fmt(p['speedup'])}" for p in report["speedup_curve"]])
    rows = ["plan,side,bucket_lo,bucket_hi,tokens_to_verify,top_k,draft_depth,memory_units"]
    for plan in ("bucketed", "vanilla"):
        for e in report["capture_comparison"].get(plan, {}).get("entries", []):
            rows.append(",".join([plan, e["side"], str(e["bucket_lo"]), str(e["bucket_hi"]),
                                  str(e["tokens_to_verify"]), str(e["top_k"]), str(e["draft_depth"]),
                                  _fmt(e["memory_units"])]))
    w("capture_memory.csv", rows)
    rows = ["arm,draft_depth,top_k,tokens_to_verify,sample,reward,mean_accept"]
    for a, arm in enumerate(report["mab_state"]["arms"]):
        st = arm["strategy"]
        for i, (r, acc) in enumerate(zip(arm["rewards"], arm["accept_lens"])):
            rows.append(",".join([str(a), str(st["draft_depth"]), str(st["top_k"]), str(st["tokens_to_verify"]),
                                  str(i), _fmt(r), _fmt(acc)]))
    w("reward_trace.csv", rows)
    return written
