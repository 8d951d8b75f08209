"""run_experiment / emit_report harness (reference
experiment.hpp:104-371 config schema, :417-424 percentile, :741-832 emission).
CPU: config parsing / validation with field-path errors, the RngStream-driven
workload helpers against the reference's own code, byte-stable CSV emission.
GPU: a short tiny-model experiment (greedy, both arms on the same requests,
SD tokens == baseline tokens, report sections present)."""
import ctypes as C
import os

import pytest

import oracle as O
from paper_2511_16665_b200 import experiment as X
from paper_2511_16665_b200.engine import ConfigError, Rng


def test_config_defaults_and_unknown_keys():
    c = X.config_from_json({})
    assert c["strategies"] == [list(s) for s in X.DEFAULT_STRATEGIES]
    assert c["mab"]["thresholds"] == [1, 2, 8, 16] and c["workload"]["requests_per_step"] == 64
    c = X.config_from_json({"rl_steps": 2, "workload": {"max_len": 64}})
    assert c["rl_steps"] == 2 and c["workload"]["max_len"] == 64 and c["workload"]["mu"] == 5.2
    with pytest.raises(ConfigError, match="workload.bogus: unknown key"):
        X.config_from_json({"workload": {"bogus": 1}})
    with pytest.raises(ConfigError, match="bogus: unknown key"):
        X.config_from_json({"bogus": 1})
    with pytest.raises(ConfigError, match="rl_steps"):
        X.config_from_json({"rl_steps": 0})
    with pytest.raises(ConfigError, match="temperature"):
        X.config_from_json({"mode": "stochastic_linear"})
    with pytest.raises(ConfigError, match="cost_model.mem_bw"):
        X.config_from_json({"cost": {"mem_bw": 0}})


def test_percentile_matches_reference_rule():
    assert X._percentile([], 0.5) == 0
    assert X._percentile([5], 0.5) == 5
    assert X._percentile([4, 1, 3, 2], 0.5) == 2   # rank ceil(0.5*4) = 2
    assert X._percentile([4, 1, 3, 2], 0.75) == 3
    assert X._percentile(list(range(1, 11)), 0.75) == 8


@pytest.mark.skipif(not O.ref_available(), reason="reference bridge not built")
def test_response_lengths_match_reference():
    """sample_response_length over the product RngStream == the reference
    (rollout.hpp:42-50) over its own RngStream, same forks."""
    R = O.ref()
    if not hasattr(R, "ref_sample_response_length"):
        pytest.skip("bridge lacks ref_sample_response_length")
    R.ref_sample_response_length.argtypes = [C.c_double, C.c_double, C.c_int, C.c_void_p]
    for seed, mu, sigma, ml in [(42, 5.2, 1.0, 1024), (7, 7.3, 1.0, 8192), (3, 2.0, 0.0, 4), (1, 0.0, 2.5, 100)]:
        r = R.ref_rng_fork(R.ref_rng_create(seed, 0), 100)
        p = Rng(seed, 0).fork(100)
        for _ in range(300):
            assert X.sample_response_length(mu, sigma, ml, p) == R.ref_sample_response_length(mu, sigma, ml, r)


def test_rng_uniform_int_and_ids():
    r = Rng(5, 0).fork(200)
    seed, stream = r.ids()
    assert seed == 5 and stream != 0
    a = Rng(5, stream)
    assert [r.uniform_int(4094) for _ in range(50)] == [a.uniform_int(4094) for _ in range(50)]


def _fake_report():
    return {
        "steps": [{"step": 0, "baseline_time": 10.5, "tlt_time": 4.25, "speedup": 10.5 / 4.25, "mean_len": 100.0,
                   "p50_len": 90, "p75_len": 120, "max_len": 300, "mean_accept": 3.1234567890123,
                   "sd_steps": 5, "plain_steps": 7, "verify_events": 40, "ngram_verify_events": 0,
                   "drafter_version": 0, "match_rate": 0.0, "training_iterations": 0}],
        "accept_rate_by_position": [0.9, 0.5, 1 / 3],
        "speedup_curve": [{"batch": 1, "tokens_to_verify": 64, "speedup": 3.6}],
        "capture_comparison": {"bucketed": {"entries": [{"side": "TARGET", "bucket_lo": 1, "bucket_hi": 1,
                                                         "tokens_to_verify": 64, "top_k": 0, "draft_depth": 0,
                                                         "memory_units": 64.0}]}},
        "mab_state": {"arms": [{"strategy": {"draft_depth": 10, "top_k": 8, "tokens_to_verify": 64},
                                "rewards": [1.5, 2.0], "accept_lens": [3.0, 4.0]}]},
    }


def test_emit_report_csv_is_byte_stable(tmp_path):
    rep = _fake_report()
    a = X.emit_report(rep, "csv", str(tmp_path / "a"))
    b = X.emit_report(rep, "csv", str(tmp_path / "b"))
    assert a == b == ["steps.csv", "accept_position.csv", "speedup_vs_batch.csv", "capture_memory.csv",
                      "reward_trace.csv"]
    for f in a:
        assert open(tmp_path / "a" / f, "rb").read() == open(tmp_path / "b" / f, "rb").read()
    steps = open(tmp_path / "a" / "steps.csv").read().splitlines()
    assert steps[0].startswith("step,baseline_time,tlt_time,speedup")
    assert steps[1].split(",")[3] == "%.12g" % (10.5 / 4.25)
    assert open(tmp_path / "a" / "accept_position.csv").read().splitlines()[3] == "3,%.12g" % (1 / 3)
    assert X.emit_report(rep, "json", str(tmp_path / "j")) == ["report.json"]
    with pytest.raises(ConfigError):
        X.emit_report(rep, "xml", str(tmp_path / "x"))


@pytest.mark.gpu
def test_gpu_run_experiment_tiny(tmp_path):
    cfg = {"rl_steps": 2, "workload": {"requests_per_step": 12, "max_len": 64, "mu": 3.5, "prompt_len": 8},
           "speedup_curve": {"batches": [1, 4], "ctx": 64}}
    rep = X.run_experiment(cfg, keep_tokens=True)
    from parity_util import greedy_streams_agree, tiny_oracle_model
    m = tiny_oracle_model()
    try:
        for st in rep["_tokens"]:
            for p, a, b in zip(st["prompts"], st["tlt"], st["baseline"]):
                ok, k, margin = greedy_streams_agree(m, p, a, b, 4096)
                assert ok, (k, margin)
    finally:
        O.orc().orc_model_destroy(m)
    rep.pop("_tokens")
    assert len(rep["steps"]) == 2
    for s in rep["steps"]:
        assert s["tokens_match"] in (True, False)  # near-tie divergences are checked against the oracle above
        assert s["sd_steps"] > 0 and s["speedup"] > 0
        assert sum(s["mab_selections"]) > 0
    assert rep["aggregate_speedup"] > 0
    assert 0 < rep["accept_rate_by_position"][0] <= 1
    cc = rep["capture_comparison"]
    assert cc["ratio"] > 1 and cc["device_bytes"]["vanilla_graphs"] > cc["device_bytes"]["bucketed_graphs"]
    assert all("measured" in p for p in rep["speedup_curve"])
    files = X.emit_report(rep, "csv", str(tmp_path))
    assert all(os.path.getsize(tmp_path / f) > 0 for f in files)
    X.emit_report(rep, "json", str(tmp_path))
