"""Host-side accounting of the MarginGate metrics (pure Python, no GPU).

Definitions follow the paper; each function cites its passage.  These are
harness logic on top of the step records the C-ABI returns; none of the
hot path runs here.
"""
from __future__ import annotations

import math
from typing import Iterable, Sequence


def latency_increment(t_method: float, t_bf16: float) -> float:
    """Overhead over BF16, PAPER.md:251 ("overhead over BF16"):
    inc = T_method / T_BF16 - 1."""
    return t_method / t_bf16 - 1.0


def increment_ratio(inc_always_on: float, inc_margingate: float) -> float:
    """"reducing LLM-42's latency increment by 2.23x":
    ratio = inc_AO / inc_MG."""
    if inc_margingate <= 0:
        return math.inf
    return inc_always_on / inc_margingate


def pert_tau(eps: Iterable[float]) -> float:
    """App. A: pert. tau = 2 * max(eps_pert)."""
    return 2.0 * max(eps)


def eps_pert(batched_logits: Sequence[float], ref_logits: Sequence[float], topk: int = 50) -> float:
    """App. A: eps = |l^{bs=N} - l^{ref}|_inf over the
    protected request's top-50 logits (index set from the reference run,
    SPEC.md:571)."""
    idx = sorted(range(len(ref_logits)), key=lambda j: (-ref_logits[j], j))[:topk]
    return max(abs(float(batched_logits[j]) - float(ref_logits[j])) for j in idx)


def tau100(rows: Sequence[tuple[float, float]]) -> float | None:
    """the smallest tested threshold whose sequence
    determinism is 100%.  rows = [(tau, seq_det in [0,1]), ...]."""
    ok = [t for t, det in rows if det >= 1.0]
    return min(ok) if ok else None


def first_divergence(batched: Sequence[int], reference: Sequence[int]) -> int | None:
    """first position where the two runs emit different tokens
    (length mismatch diverges at the first missing position)."""
    n = min(len(batched), len(reference))
    for i in range(n):
        if batched[i] != reference[i]:
            return i
    return None if len(batched) == len(reference) else n


def synchronous_samples(batched: Sequence[int], reference: Sequence[int]) -> tuple[int, int]:
    """(synchronous samples, divergence events) of one trial, PAPER.md:42:
    positions up to and including the first divergence."""
    d = first_divergence(batched, reference)
    if d is None:
        return len(reference), 0
    return d + 1, 1


def flip_rate(trials: Iterable[tuple[Sequence[int], Sequence[int]]]) -> float:
    """Synchronous flip rate (tab:flip_rate): sum of divergence
    events / sum of synchronous samples."""
    s = e = 0
    for b, r in trials:
        ss, ee = synchronous_samples(b, r)
        s += ss
        e += ee
    if s == 0:
        raise ValueError("no synchronous samples")
    return e / s


def margin_recall(event_margins: Sequence[float], tau: float) -> float:
    """App. C: fraction of divergence events whose margin
    is below tau (strict, as the gate)."""
    if not event_margins:
        raise ValueError("no divergence events")
    return sum(1 for g in event_margins if g < tau) / len(event_margins)


def seq_determinism(seqs: Sequence[Sequence[int]], refs: Sequence[Sequence[int]]) -> float:
    """a run is sequence-deterministic when its complete
    decoded sequence is identical to the reference."""
    assert len(seqs) == len(refs)
    return sum(1 for a, b in zip(seqs, refs) if list(a) == list(b)) / len(seqs)


def rates(stats: dict) -> dict:
    """r_verify and r_repair, over protected decode steps."""
    p = stats.get("protected_rows", 0)
    return {
        "r_verify": stats["triggers"] / p if p else 0.0,
        "r_repair": stats["repairs"] / p if p else 0.0,
    }


def kv_deviation(batched_cols, ref_cols):
    """S2.2 Observation 2: E^K_p = ||K^{bs=N}_{:,p,:} - K^{ref}_{:,p,:}||_2
    and E^V_p likewise, per layer and position.  Inputs: per position p a
    bf16 column [L][2 (K, V)][KV][hd] (uint16 bit patterns, as
    mgd_read_column returns them).  Returns (EK, EV) float64 arrays [P][L]."""
    import numpy as np
    a = np.asarray(batched_cols, dtype=np.uint16).astype(np.uint32) << 16
    b = np.asarray(ref_cols, dtype=np.uint16).astype(np.uint32) << 16
    d = a.view(np.float32).astype(np.float64) - b.view(np.float32).astype(np.float64)
    e = np.sqrt((d * d).sum(axis=(-2, -1)))        # [P][L][2]
    return e[..., 0], e[..., 1]


def divergence_aligned(err, p0: int, p_div):
    """Fig. fig:err_vs_dist: per offset Delta = p - p_div the
    deviation; positions are p0 + index.  Without a divergence, Delta is None."""
    out = {}
    for i, row in enumerate(err):
        delta = None if p_div is None else p0 + i - p_div
        out.setdefault(delta, []).append(row)
    return out
