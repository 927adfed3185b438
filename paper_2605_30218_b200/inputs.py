"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method: only model SHAPES (public HF
configs of the models PAPER.md:51-55 names, re-checked per SURVEY 2.3), the
weight seed, and seeded prompt / protection-mask generators.  Both the CUDA
path and the oracle consume these as plain inputs (DESIGN.md section 5,
"input recipe").  It imports nothing from the rest of the package.
"""
from __future__ import annotations

import numpy as np

WEIGHT_SEED = 42  # "Weights use seed 42"

# Model shapes.  [public cfg] for the three named models; "tiny" is
# BASELINE.json configs[0] (d_ff and KV heads are builder choices, SURVEY
# 8(d)); "wide" is the wide-shallow parity config of SURVEY 4 (8B widths,
# 2 layers, full vocabulary).
SHAPES = {
    "tiny": dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=4, head_dim=64, d_ff=1024, vocab=4096,
                 qkv_bias=0, rms_eps=1e-5, rope_theta=10000.0),
    "tiny_gqa": dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=2, head_dim=64, d_ff=1024, vocab=4096,
                     qkv_bias=1, rms_eps=1e-6, rope_theta=1000000.0),
    "wide": dict(n_layers=2, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, d_ff=14336, vocab=128256,
                 qkv_bias=0, rms_eps=1e-5, rope_theta=500000.0),
    # long-context parity configs (tests/test_gpu_longctx.py): the attention
    # shapes of Llama-3.1-8B (32 q / 8 kv heads, hd 128) and of
    # DSR1-Distill-Qwen-7B (28 / 4, hd 128, qkv bias) on narrow, shallow
    # models, so the oracle can recompute contexts of 500-4000 keys
    "longattn": dict(n_layers=2, d_model=1024, n_heads=32, n_kv_heads=8, head_dim=128, d_ff=2048, vocab=16384,
                     qkv_bias=0, rms_eps=1e-5, rope_theta=500000.0),
    "dsr1attn": dict(n_layers=2, d_model=896, n_heads=28, n_kv_heads=4, head_dim=128, d_ff=2048, vocab=16384,
                     qkv_bias=1, rms_eps=1e-6, rope_theta=10000.0),
    "llama8b": dict(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, d_ff=14336,
                    vocab=128256, qkv_bias=0, rms_eps=1e-5, rope_theta=500000.0),
    "qwen14b": dict(n_layers=48, d_model=5120, n_heads=40, n_kv_heads=8, head_dim=128, d_ff=13824,
                    vocab=152064, qkv_bias=1, rms_eps=1e-6, rope_theta=1000000.0),
    "dsr1_7b": dict(n_layers=28, d_model=3584, n_heads=28, n_kv_heads=4, head_dim=128, d_ff=18944,
                    vocab=152064, qkv_bias=1, rms_eps=1e-6, rope_theta=10000.0),
}

# Decode-length shapes: (prompt_len, decode_len).
WORKLOADS = {
    "math500": (128, 512),
    "gsm8k": (128, 256),
    "humaneval": (160, 448),
    "dsr1_long": (128, 4096),
}


def shape(name: str, seed: int = WEIGHT_SEED) -> dict:
    s = dict(SHAPES[name])
    s["weight_seed"] = seed
    s["name"] = name
    return s


def prompts(n: int, lengths, vocab: int, seed: int = 7) -> list[list[int]]:
    """Uniform-random token ids, request i drawn from seed + i.
    `lengths` is an int or a list of per-request lengths."""
    if isinstance(lengths, int):
        lengths = [lengths] * n
    out = []
    for i in range(n):
        rng = np.random.default_rng(seed + i)
        out.append([int(t) for t in rng.integers(0, vocab, size=int(lengths[i]))])
    return out


def ragged_lengths(n: int, lo: int, hi: int, seed: int = 11) -> list[int]:
    """Lengths in [lo, hi] (BASELINE configs[0]: 8..23 crosses 16-token pages)."""
    rng = np.random.default_rng(seed)
    return [int(x) for x in rng.integers(lo, hi + 1, size=n)]


def protected_mask(B: int, mode: str = "all", seed: int = 3) -> np.ndarray:
    """'all' rows protected, 'one' (row 0, the paper's protocol PAPER.md:42),
    'none', or 'half' (seeded random half)."""
    if mode == "all":
        return np.ones(B, np.uint8)
    if mode == "none":
        return np.zeros(B, np.uint8)
    if mode == "one":
        m = np.zeros(B, np.uint8)
        m[0] = 1
        return m
    rng = np.random.default_rng(seed)
    return (rng.random(B) < 0.5).astype(np.uint8)
