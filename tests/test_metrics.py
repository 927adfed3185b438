"""Host-side metric arithmetic pinned to values the paper prints
(tests/golden/paper_values.json, each entry cited)."""
import json
import math
import os

import pytest

from paper_2605_30218_b200 import metrics

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


@pytest.mark.parametrize("row", GOLD["headline_ratio"])
def test_headline_ratio(row):
    # PAPER.md:5 "reducing LLM-42's latency increment by 2.23x/1.99x"
    r = metrics.increment_ratio(row["llm42_overhead_pct"] / 100, row["margingate_overhead_pct"] / 100)
    assert round(r, 2) == row["ratio"]


@pytest.mark.parametrize("name", ["Llama-3.1-8B", "Qwen2.5-14B"])
def test_latency_increment_from_walltimes(name):
    w = GOLD["walltime_bs8_s"][name]
    t_llm42 = w["bf16"] * (1 + w["llm42_pct"] / 100)
    assert metrics.latency_increment(t_llm42, w["bf16"]) == pytest.approx(w["llm42_pct"] / 100)


@pytest.mark.parametrize("row", GOLD["eps_pert_exact_rows"])
def test_pert_tau(row):
    # tab:eps_pert: "pert. tau is 2*max(eps_pert)"
    assert metrics.pert_tau([0.1, row["max_eps"], 0.3]) == pytest.approx(row["pert_tau"])


@pytest.mark.parametrize("key", ["pareto_llama8b", "pareto_dsr1", "pareto_qwen14b"])
def test_tau100_selection(key):
    blk = GOLD[key]
    assert metrics.tau100([tuple(r) for r in blk["rows"]]) == blk["tau100"]
    assert metrics.tau100([(1.0, 0.5)]) is None


def test_eps_pert_topk_window():
    ref = [float(i) for i in range(100)]
    bat = list(ref)
    bat[0] += 5.0        # outside the reference top-50: ignored
    bat[99] += 0.25      # inside
    assert metrics.eps_pert(bat, ref, 50) == 0.25


def test_flip_rate_and_divergence():
    ex = GOLD["spec_examples"]["flip_rate"]
    trials = [([1, 2, 3, 4], [1, 2, 3, 4]), ([1, 9, 3, 4], [1, 2, 3, 4])]
    assert metrics.flip_rate(trials) == pytest.approx(ex["value"])
    assert metrics.first_divergence([1, 2], [1, 2, 3]) == 2
    assert metrics.first_divergence([1, 2, 3], [1, 2, 3]) is None
    assert metrics.first_divergence([0, 2], [1, 2]) == 0


def test_margin_recall():
    ex = GOLD["spec_examples"]["recall"]
    assert metrics.margin_recall(ex["margins"], ex["tau"]) == pytest.approx(ex["value"])
    assert metrics.margin_recall(ex["margins"], math.inf) == 1.0
    assert metrics.margin_recall(ex["margins"], 0.0) == 0.0


def test_seq_determinism_and_rates():
    assert metrics.seq_determinism([[1, 2], [1, 3]], [[1, 2], [1, 2]]) == 0.5
    r = metrics.rates({"triggers": 10, "repairs": 2, "protected_rows": 40})
    assert r == {"r_verify": 0.25, "r_repair": 0.05}


def test_kv_deviation_closed_form():
    """E^K_p / E^V_p: identical columns give 0; one element off
    by a known bf16 difference gives exactly that L2 norm, in its own layer,
    position and K/V slot only; sqrt of a sum over heads and dims."""
    import numpy as np
    L, KV, hd, P = 3, 2, 4, 5
    rng = np.random.default_rng(0)
    base = (rng.integers(0x3F00, 0x4000, size=(P, L, 2, KV, hd))).astype(np.uint16)
    ek, ev = metrics.kv_deviation(base, base)
    assert ek.shape == (P, L) and not ek.any() and not ev.any()
    other = base.copy()
    other[2, 1, 1, 0, 3] = 0x3F80            # 1.0
    other[2, 1, 1, 1, 0] = 0x4000            # 2.0
    a = base.astype(np.uint32) << 16
    x = a.view(np.float32).astype(np.float64)
    want = np.sqrt((x[2, 1, 1, 0, 3] - 1.0) ** 2 + (x[2, 1, 1, 1, 0] - 2.0) ** 2)
    ek, ev = metrics.kv_deviation(base, other)
    assert not ek.any()
    assert ev[2, 1] == pytest.approx(want, rel=1e-12) and np.count_nonzero(ev) == 1
    al = metrics.divergence_aligned(ev, 10, 12)
    assert sorted(al) == [-2, -1, 0, 1, 2] and al[0][0][1] == ev[2, 1]
