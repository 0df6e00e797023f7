"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic (no scales, no codes, no
GEMM).  It only draws random numbers and rounds them to the storage dtype of
the inputs (bf16 / fp16 bit patterns), so that the oracle (`oracle/`) and the
product path (`paper_2308_09723_b200/`) consume the very same bytes.

Input recipe (following SURVEY.md §8(d)):
  * weights W[N, K] ~ N(0, 0.02^2): "generally exhibit a normal distribution
    centered around zero" (§3.1);
  * outlier variant: one planted +-magnitude entry per selected matrix
    ("outliers can distort the weight distribution");
  * activations A[M, K] ~ N(0, 1) (zero-mean keeps the 2e-3 tolerance
    meaningful, SURVEY.md §8(c) "GEMM tolerance feasibility");
  * seeds: W 1000+matrix_id, A 2000+config_id, routing 3000.
All generators use numpy PCG64 (`np.random.default_rng(seed)`).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "f32_to_bf16_bits",
    "f32_to_fp16_bits",
    "gaussian_bits",
    "gaussian_with_outliers_bits",
    "activations_bits",
    "zipf_routing",
    "uniform_routing",
]


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float32 values to bf16 (round-to-nearest-even) and return uint16 bit patterns.

    Storage-format conversion of generated inputs only (not method arithmetic).
    NaN is not produced by the generators.
    """
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = (u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)
    return r.astype(np.uint16)


def f32_to_fp16_bits(x: np.ndarray) -> np.ndarray:
    """Round float32 values to IEEE fp16 (numpy's RNE cast) and return uint16 bit patterns."""
    return np.ascontiguousarray(x, dtype=np.float32).astype(np.float16).view(np.uint16)


def _to_bits(x32: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return f32_to_bf16_bits(x32)
    if dtype == "fp16":
        return f32_to_fp16_bits(x32)
    if dtype == "fp32":
        return np.ascontiguousarray(x32, dtype=np.float32).view(np.uint32)
    raise ValueError(f"unknown dtype {dtype}")


def gaussian_bits(shape, std: float, seed: int, dtype: str = "bf16", mean: float = 0.0) -> np.ndarray:
    """N(mean, std^2) samples drawn as float32 with PCG64(seed), stored as `dtype` bit patterns."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(size=shape, dtype=np.float32) * np.float32(std) + np.float32(mean)
    return _to_bits(x, dtype)


def gaussian_with_outliers_bits(shape, std: float, seed: int, outlier_count: int = 1,
                                outlier_magnitude: float = 1.0, dtype: str = "bf16") -> np.ndarray:
    """Gaussian weights with exactly `outlier_count` entries set to +-outlier_magnitude at
    seeded positions (SPEC.md:52-60 `gaussian_with_outliers`)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(size=shape, dtype=np.float32) * np.float32(std)
    flat = x.reshape(-1)
    pos = rng.choice(flat.size, size=outlier_count, replace=False)
    sign = np.where(rng.integers(0, 2, size=outlier_count) == 0, -1.0, 1.0).astype(np.float32)
    flat[pos] = sign * np.float32(outlier_magnitude)
    return _to_bits(x, dtype)


def activations_bits(M: int, K: int, seed: int, dtype: str = "bf16", std: float = 1.0) -> np.ndarray:
    """Activation matrix A[M, K] ~ N(0, std^2) as `dtype` bit patterns."""
    return gaussian_bits((M, K), std, seed, dtype)


def wide_range_activations_bits(M: int, K: int, seed: int, dtype: str = "bf16",
                                log2_lo: float = -60.0, log2_hi: float = 60.0,
                                token_shift: int = 30) -> np.ndarray:
    """A[M, K] with log-uniform magnitudes 2^U(log2_lo, log2_hi), random signs, and per-token
    structure: token m's magnitudes are additionally shifted by a per-token power of two, every
    4th token has one all-zero 128-column chunk, and one token is entirely zero."""
    rng = np.random.default_rng(seed)
    e = rng.uniform(log2_lo, log2_hi, size=(M, K))
    e += rng.integers(-token_shift, token_shift + 1, size=(M, 1))
    x = np.sign(rng.standard_normal((M, K))) * np.exp2(e)
    for m in range(0, M, 4):
        c = int(rng.integers(0, max(1, K // 128)))
        x[m, c * 128:(c + 1) * 128] = 0.0
    if M > 2:
        x[M // 2] = 0.0
    return _to_bits(x.astype(np.float32), dtype)


def uniform_routing(E: int, tokens_per_expert: int) -> np.ndarray:
    """Expert offsets [E+1] for a uniform routing with `tokens_per_expert` tokens each."""
    return np.arange(E + 1, dtype=np.int64) * int(tokens_per_expert)


def zipf_routing(E: int, total_tokens: int, seed: int = 3000, s: float = 1.0) -> np.ndarray:
    """Expert offsets [E+1] for a Zipf(s) skewed routing of `total_tokens` tokens.

    Tokens are split by a multinomial with p_e ∝ 1/rank_e^s where the ranks are a
    seeded permutation of 1..E (MoE routing detail).
    """
    rng = np.random.default_rng(seed)
    ranks = rng.permutation(E) + 1
    p = 1.0 / ranks.astype(np.float64) ** s
    p /= p.sum()
    counts = rng.multinomial(total_tokens, p)
    off = np.zeros(E + 1, dtype=np.int64)
    off[1:] = np.cumsum(counts)
    return off


def gaussian_torch(shape, std: float, seed: int, device="cuda", dtype=None):
    """Large-input generator (full-size configs): N(0, std^2) drawn on `device` with a seeded
    torch.Generator (Philox), rounded to `dtype` (default bf16).  Used where numpy generation of
    ~6e8 values would dominate test time; the oracle consumes the same bytes copied back."""
    import torch
    g = torch.Generator(device=device).manual_seed(int(seed))
    x = torch.randn(*shape, generator=g, device=device, dtype=torch.float32) * float(std)
    return x.to(dtype or torch.bfloat16)
