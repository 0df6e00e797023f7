"""CPU oracle for the FineQuant hot path (arXiv 2308.09723).

*** TEST INFRASTRUCTURE ONLY. ***
Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this module.  The product path
(`paper_2308_09723_b200/`) never imports it and shares no code with it.

Plain, slow, obviously-correct numpy in float64.  Every function cites the
passage it follows (PAPER.md line, section).  Readings where the paper is
silent/ambiguous are the ones listed in DESIGN.md §2 (R1..R12) and follow
SURVEY.md §8(c).

Parity status per function (see DESIGN.md §2 and tests/test_oracle_*.py):
  decode_*, round_to_format, encode_format ........ pinned (exhaustive vs numpy/IEEE casts, hand values)
  scale_for_amax, quantize ........................ pinned (hand example tests/golden/quant_hand.txt,
                                                    exact round-trip construction, error-bound invariants,
                                                    exact-rational brute force)
  pack_codes / unpack_codes ....................... pinned (hand bytes 0xC2 0x86, round-trip law)
  pack_bitstream / unpack_bitstream (int3/int2) ... pinned (hand-packed int3 bytes tests/golden/int3_hand.txt,
                                                    equals the independent int4/int8 packers at b=4/8,
                                                    round-trip law)
  quantize_acts_i8 / quantize_intscale / gemm_i8 .. pinned (hand-worked tests/golden/intscale_hand.txt,
  (int8-activation x int4-weight, integer scales)   exact round-trip construction, numpy float32 IEEE
                                                    division, exact-rational brute force, invariants)
  adapt_ladder / adapt_group_size ................. pinned on SPEC fixtures + invariants only;
                                                    paper parity UNPINNED (the paper prints no
                                                    worked example and its inequality is ambiguous, R6)
  gemm / rel_err .................................. pinned (integer-exact special case, one-hot / identity,
                                                    linearity, pure-Python brute force)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------------------------
# Storage formats.  A format is (significand bits incl. the implicit one, min normal exponent,
# max finite value).  bf16: 8 / -126;  fp16: 11 / -14;  fp32: 24 / -126.
# ----------------------------------------------------------------------------------------------


@dataclass(frozen=True)
class Fmt:
    name: str
    p: int
    emin: int
    max_finite: float


BF16 = Fmt("bf16", 8, -126, float.fromhex("0x1.fep127"))
FP16 = Fmt("fp16", 11, -14, 65504.0)
FP32 = Fmt("fp32", 24, -126, float.fromhex("0x1.fffffep127"))
FORMATS = {"bf16": BF16, "fp16": FP16, "fp32": FP32}


def decode_bits(bits: np.ndarray, fmt: str) -> np.ndarray:
    """Interpret stored bit patterns of `fmt` as exact float64 values."""
    bits = np.asarray(bits)
    if fmt == "bf16":
        return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)
    if fmt == "fp16":
        return bits.astype(np.uint16).view(np.float16).astype(np.float64)
    if fmt == "fp32":
        return bits.astype(np.uint32).view(np.float32).astype(np.float64)
    raise ValueError(fmt)


def round_to_format(x: np.ndarray, fmt: Fmt) -> np.ndarray:
    """Round float64 values to the nearest value of `fmt`, ties to even, in ONE rounding step.

    |x| = m * 2^e (frexp, m in [0.5,1)); the quantum is 2^(E-(p-1)) with E = max(e-1, emin)
    (the max handles subnormals).  |x|/quantum is exact in float64, np.rint rounds it
    half-to-even exactly, and the product is exact.  Values beyond the largest finite value
    (after rounding) become +-inf (IEEE overflow under RNE).
    """
    x = np.asarray(x, dtype=np.float64)
    ax = np.abs(x)
    _, e = np.frexp(ax)
    E = np.maximum(e - 1, fmt.emin)
    q = np.ldexp(1.0, E - (fmt.p - 1))
    r = np.rint(ax / q) * q
    r = np.where(ax == 0, 0.0, r)
    r = np.where(r > fmt.max_finite, np.inf, r)
    return np.copysign(r, x)


def encode_format(v: np.ndarray, fmt: Fmt) -> np.ndarray:
    """Bit patterns of values that are already exactly representable in `fmt`."""
    v = np.asarray(v, dtype=np.float64)
    if fmt is BF16:
        f = v.astype(np.float32)  # exact: v is a bf16 value, hence an fp32 value
        assert np.all((f.astype(np.float64) == v) | np.isnan(v))
        return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)
    if fmt is FP16:
        h = v.astype(np.float16)
        assert np.all((h.astype(np.float64) == v) | np.isnan(v))
        return h.view(np.uint16)
    if fmt is FP32:
        return v.astype(np.float32).view(np.uint32)
    raise ValueError(fmt)


# ----------------------------------------------------------------------------------------------
# Quantization: linear absmax, symmetric, group-wise (App. A; group-wise
# generalisation PAPER.md:179 §4.1 "each contiguous block of B elements in a given column has its
# own scaling factor"; scales in the activation dtype PAPER.md:170 §4.1).
# ----------------------------------------------------------------------------------------------


def round_half_away(y: np.ndarray) -> np.ndarray:
    """integer(.) of App. A, read as round half away from zero (reading R1).

    Exact for float64 y: trunc and the fractional part y - trunc(y) are exact.
    """
    y = np.asarray(y, dtype=np.float64)
    t = np.trunc(y)
    frac = y - t
    return t + np.sign(y) * (np.abs(frac) >= 0.5)


def scale_for_amax(amax: np.ndarray, bits: int, scale_fmt: Fmt) -> np.ndarray:
    """s = 2 * max|A_group| / (2^b - 1)   (App. A), stored in `scale_fmt`
    (reading R3: the activation dtype) with one round-to-nearest-even (reading R4).

    The float64 quotient is the correctly rounded exact quotient; it can never sit on a
    bf16/fp16 rounding tie (the exact value m*2^e/(2^b-1) has a periodic non-zero binary
    expansion, R4), so rounding it once more equals rounding the exact rational.
    """
    amax = np.asarray(amax, dtype=np.float64)
    return round_to_format(2.0 * amax / float((1 << bits) - 1), scale_fmt)


def group_amax(W: np.ndarray, group: int) -> np.ndarray:
    """amax[j, n] = max_{k in group j} |W[n, k]|   for W stored [N, K] (paper column n = row n)."""
    N, K = W.shape
    G = K // group
    return np.abs(W).reshape(N, G, group).max(axis=2).T.copy()


@dataclass
class QuantResult:
    q: np.ndarray          # int8 [N, K] codes
    s: np.ndarray          # float64 [G, N] scales (values of scale_fmt)
    s_bits: np.ndarray     # uint16 [G, N] stored scale bit patterns
    status: int            # 0 ok; 1 non-finite input; 2 scale overflow


def quantize(W: np.ndarray, bits: int, group: int, scale_fmt: Fmt = BF16) -> QuantResult:
    """Group-wise linear absmax quantization of W[N, K] (paper column n stored as row n).

    Steps:
      1. x = W[n, k] exactly (float64);          non-finite -> status 1, group codes/scale 0
      2. amax per (group j, column n)
      3. s = RNE_fmt(2*amax/(2^b-1))            (App. A)
      4. s == 0 -> codes 0                       (reading R5)
      5. q = clamp(integer(x / s), -2^(b-1), 2^(b-1)-1)   (App. A; R1/R2)
    """
    W = np.asarray(W, dtype=np.float64)
    N, K = W.shape
    if bits not in (2, 3, 4, 5, 6, 7, 8):
        raise ValueError("bits")
    if group <= 0 or K % group:
        raise ValueError("group must divide K")
    G = K // group
    finite = np.isfinite(W).reshape(N, G, group).all(axis=2).T  # [G, N]
    Wz = np.where(np.isfinite(W), W, 0.0)
    amax = group_amax(Wz, group)
    s = scale_for_amax(amax, bits, scale_fmt)
    status = 0
    if not finite.all():
        status = 1
    over = ~np.isfinite(s)
    if over.any():
        status = status or 2
    bad = (~finite) | over
    s = np.where(bad, 0.0, s)
    s_full = np.repeat(s.T, group, axis=1)  # [N, K]
    with np.errstate(divide="ignore", invalid="ignore"):
        y = np.where(s_full > 0, Wz / np.where(s_full > 0, s_full, 1.0), 0.0)
    lo, hi = -(1 << (bits - 1)), (1 << (bits - 1)) - 1
    q = np.clip(round_half_away(y), lo, hi).astype(np.int8)
    return QuantResult(q=q, s=s, s_bits=encode_format(s, scale_fmt), status=status)


def dequantize(q: np.ndarray, s: np.ndarray, group: int) -> np.ndarray:
    """A'[n, k] = Q[n, k] * s[k // group, n]   (App. A), exact in float64."""
    q = np.asarray(q, dtype=np.float64)
    return q * np.repeat(np.asarray(s, dtype=np.float64).T, group, axis=1)


# ----------------------------------------------------------------------------------------------
# Packing (canonical layout): codes[N, K*b/8], K contiguous per column n;
# int4 byte (n, k/2) = (q[n,k] & 0xF) | (q[n,k+1] & 0xF) << 4 (low nibble first);
# int8 byte = two's complement q.
# ----------------------------------------------------------------------------------------------


def pack_codes(q: np.ndarray, bits: int) -> np.ndarray:
    q = np.asarray(q).astype(np.int16)
    N, K = q.shape
    if bits == 8:
        return (q & 0xFF).astype(np.uint8)
    if bits == 4:
        assert K % 2 == 0
        lo = (q[:, 0::2] & 0xF).astype(np.uint8)
        hi = (q[:, 1::2] & 0xF).astype(np.uint8)
        return (lo | (hi << 4)).astype(np.uint8)
    if bits in (2, 3):
        return pack_bitstream(q, bits)
    raise ValueError("bits")


def unpack_codes(codes: np.ndarray, bits: int, K: int) -> np.ndarray:
    codes = np.asarray(codes, dtype=np.uint8)
    N = codes.shape[0]
    if bits == 8:
        return codes.view(np.int8).reshape(N, K).copy()
    if bits == 4:
        lo = (codes & 0xF).astype(np.int16)
        hi = (codes >> 4).astype(np.int16)
        lo = np.where(lo >= 8, lo - 16, lo)
        hi = np.where(hi >= 8, hi - 16, hi)
        out = np.empty((N, K), dtype=np.int8)
        out[:, 0::2] = lo
        out[:, 1::2] = hi
        return out
    if bits in (2, 3):
        return unpack_bitstream(codes, bits, K)
    raise ValueError("bits")


def pack_bitstream(q: np.ndarray, bits: int) -> np.ndarray:
    """Little-endian bit stream per column: code k of column n occupies
    bits [b*k, b*k + b) of the column's stream, least significant bit first, two's complement;
    byte i of the column = stream bits [8i, 8i + 8).  int4 / int8 are the special cases above.
    Used for the int3 / int2 codes of the paper's low-bit variants (PAPER.md:332-346,
    tab:optiml-mt), for which the paper ships no kernel and no layout.
    Requires K * bits % 8 == 0 (every column a whole number of bytes)."""
    q = np.asarray(q).astype(np.int64)
    N, K = q.shape
    assert (K * bits) % 8 == 0
    out = np.zeros((N, K * bits // 8), dtype=np.uint8)
    mask = (1 << bits) - 1
    for k in range(K):                      # plain loop over code positions, bit by bit
        f = q[:, k] & mask                  # the b-bit two's-complement field
        for b in range(bits):
            pos = bits * k + b
            out[:, pos // 8] |= (((f >> b) & 1) << (pos % 8)).astype(np.uint8)
    return out


def unpack_bitstream(codes: np.ndarray, bits: int, K: int) -> np.ndarray:
    codes = np.asarray(codes, dtype=np.uint8)
    N = codes.shape[0]
    out = np.zeros((N, K), dtype=np.int64)
    for k in range(K):
        f = np.zeros(N, dtype=np.int64)
        for b in range(bits):
            pos = bits * k + b
            f |= ((codes[:, pos // 8].astype(np.int64) >> (pos % 8)) & 1) << b
        out[:, k] = np.where(f >= (1 << (bits - 1)), f - (1 << bits), f)
    return out.astype(np.int8)


# ----------------------------------------------------------------------------------------------
# Adaptive fine-grained group size (§3.3), step by step, exhaustive:
# every group's range at every level is recomputed from W (no pyramid reuse).
# Reading R6: "halve while some child ratio < alpha; stop when all >= alpha".
# Reading R7: range = max|.|.  Reading R9: ladder halves exactly from K, g % 16 == 0, g >= min_group.
# Reading R10: alpha = alpha_milli / 1000, default 500; min_group default 16.
# Reading R11: one g per matrix.
# ----------------------------------------------------------------------------------------------


def adapt_ladder(K: int, min_group: int = 16) -> list[int]:
    """Group sizes g_0 = K, g_{L+1} = g_L / 2 while g_L even, g_L/2 >= min_group, g_L/2 % 16 == 0."""
    ladder = [K]
    g = K
    while g % 2 == 0 and g // 2 >= min_group and (g // 2) % 16 == 0:
        g //= 2
        ladder.append(g)
    return ladder


@dataclass
class AdaptLevel:
    level: int
    group: int
    min_ratio: float
    count_below: int
    flag: bool
    accepted: bool


@dataclass
class AdaptReport:
    group: int
    alpha_milli: int
    levels: list = field(default_factory=list)


def adapt_flags(W: np.ndarray, alpha_milli: int = 500, min_group: int = 16) -> list[bool]:
    """flag_L (L >= 1) = exists (n, j): range_L(n, j) < alpha * range_{L-1}(n, j // 2),
    evaluated as 1000 * child < alpha_milli * parent (exact in float64; a zero parent never fires,
    i.e. ratio := 1)."""
    return [lv.flag for lv in adapt_report(W, alpha_milli, min_group).levels]


def adapt_report(W: np.ndarray, alpha_milli: int = 500, min_group: int = 16) -> AdaptReport:
    W = np.asarray(W, dtype=np.float64)
    N, K = W.shape
    if not (1 <= alpha_milli <= 1000):
        raise ValueError("alpha_milli must be in [1, 1000]")
    ladder = adapt_ladder(K, min_group)
    rep = AdaptReport(group=K, alpha_milli=alpha_milli)
    still = True
    for L in range(1, len(ladder)):
        g_parent, g_child = ladder[L - 1], ladder[L]
        parent = group_amax(W, g_parent)           # [G_{L-1}, N], recomputed from W
        child = group_amax(W, g_child)             # [G_L, N], recomputed from W
        par_of_child = parent[np.arange(child.shape[0]) // 2, :]
        below = 1000.0 * child < float(alpha_milli) * par_of_child
        with np.errstate(divide="ignore", invalid="ignore"):
            ratio = np.where(par_of_child > 0, child / np.where(par_of_child > 0, par_of_child, 1.0), 1.0)
        flag = bool(below.any())
        accepted = still and flag
        if accepted:
            rep.group = g_child
        still = accepted
        rep.levels.append(AdaptLevel(L, g_child, float(ratio.min()), int(below.sum()), flag, accepted))
    return rep


def adapt_group_size(W: np.ndarray, alpha_milli: int = 500, min_group: int = 16) -> int:
    return adapt_report(W, alpha_milli, min_group).group


def adapt_decide(flags: list[bool], K: int, min_group: int = 16) -> int:
    """g of the last level of the accepted prefix of flags (level 0 = K is always accepted).
    TP: callers OR the flags of all shards before deciding."""
    ladder = adapt_ladder(K, min_group)
    g = K
    for L, f in enumerate(flags, start=1):
        if not f:
            break
        g = ladder[L]
    return g


# ----------------------------------------------------------------------------------------------
# GEMM (§4.1: "dequantize the weights to match the data type of the activation and
# perform floating-point tensor core math"); the result the method computes is the plain
# definition C = A . dequant(Q)^T, so the oracle is that definition in float64.
# ----------------------------------------------------------------------------------------------


def gemm(A: np.ndarray, q: np.ndarray, s: np.ndarray, group: int, cols=None):
    """C_ref[m, n] = sum_k A[m,k] * (q[n,k] * s[k//g, n])   in float64, and
    D[m, n] = sum_k |A[m,k] * q[n,k] * s[k//g, n]|   (tolerance denominator).

    `cols` optionally restricts the computation to a subset of output columns n (sampled parity).
    """
    A = np.asarray(A, dtype=np.float64)
    if cols is not None:
        cols = np.asarray(cols)
        q = np.asarray(q)[cols]
        s = np.asarray(s)[:, cols]
    Wd = dequantize(q, s, group)            # [n, K]
    C = A @ Wd.T
    D = np.abs(A) @ np.abs(Wd).T
    return C, D


def rel_err(C_test: np.ndarray, C_ref: np.ndarray, D: np.ndarray) -> float:
    """max_{m,n} |C_test - C_ref| / D, with D == 0 requiring C_test == 0 exactly (else inf)."""
    C_test = np.asarray(C_test, dtype=np.float64)
    diff = np.abs(C_test - C_ref)
    zero = D == 0
    if np.any(zero & (diff != 0)):
        return math.inf
    if np.all(zero):
        return 0.0
    return float(np.max(diff[~zero] / D[~zero]))


def gemm_grouped(A: np.ndarray, offsets: np.ndarray, experts: list, cols=None):
    """MoE expert FFN batch: rows offsets[e]:offsets[e+1] of A multiply
    expert e's dequantized weights; each expert is (q, s, group).  Returns (C, D) over all rows."""
    A = np.asarray(A, dtype=np.float64)
    N = experts[0][0].shape[0] if cols is None else len(cols)
    C = np.zeros((A.shape[0], N))
    D = np.zeros((A.shape[0], N))
    for e, (q, s, g) in enumerate(experts):
        lo, hi = int(offsets[e]), int(offsets[e + 1])
        if hi > lo:
            C[lo:hi], D[lo:hi] = gemm(A[lo:hi], q, s, g, cols)
    return C, D


# ----------------------------------------------------------------------------------------------
# int8 activations x int4 weights with INTEGER group scales -- the paper's stated future work:
# "the proposed method does not leverage integer instructions even when they are available"
# (§5) and "using int8 activations and int4 weights with integer scales for
# fine-grained quantization" (§5).  Readings (R15-R19):
#   weights: App. A's fine scale s_j = 2 amax_j / (2^b - 1) is re-expressed as
#     sigma[n] * z[j, n]: sigma = a per-column fp32 scale, z an integer in [1, Z] (Z = 16 for
#     int4: |q * z| <= 128 fits a signed byte, so dequantized weights are int8 and the whole
#     K-reduction is one exact integer dot product);
#       sigma[n] = RN_fp32( 2 * max_j amax_j / ((2^b - 1) * Z) )
#       z[j, n]  = clamp( ceil( (2 amax_j / (2^b - 1)) / sigma[n] ), 1, Z )   (effective scale >= s_j)
#       q[n, k]  = clamp( integer( W[n,k] / (sigma[n] z[j,n]) ), -2^(b-1), 2^(b-1) - 1 )
#     both decisions (ceil, integer) taken in float64 (sigma * z is exact there);
#   activations: per-token (row) symmetric int8, App. A applied to the row with b = 8 and the
#     symmetric range [-127, 127]: s_a[m] = RN_fp32(amax_m / 127),
#     a_q = clamp(integer(fp32(A / s_a)), -127, 127), the division in IEEE fp32 (the kernel's precision);
#   GEMM: acc[m, n] = sum_k a_q[m,k] * q[n,k] * z[k/g, n]  (exact integer), C = acc * s_a[m] * sigma[n].
# ----------------------------------------------------------------------------------------------

INTSCALE_Z = 16


@dataclass
class ActQuant:
    a_q: np.ndarray        # int8 [M, K]
    s_a: np.ndarray        # float64 [M] (fp32 values)
    status: int            # 0 ok; 1 non-finite input row(s) (their codes and scale are 0)
    rowsum: np.ndarray = None  # int64 [M] = sum_k a_q[m, k] (plain definition)


def quantize_acts_i8(A: np.ndarray) -> ActQuant:
    """Per-token symmetric int8 activation quantization (R17): s_a = RN_fp32(amax / 127) and
    a_q = clamp(integer(A / s_a), -127, 127) with the quotient an IEEE fp32 division (numpy float32
    arithmetic is IEEE: one correctly rounded division) and integer() = round half away (R1)."""
    A = np.asarray(A, dtype=np.float64)
    M, K = A.shape
    fin = np.isfinite(A).all(axis=1)
    Az = np.where(fin[:, None], A, 0.0)
    amax = np.abs(Az).max(axis=1) if K else np.zeros(M)
    # amax / 127 has a periodic binary expansion (period 7) unless exact, so the float64 quotient
    # is never an fp32 rounding midpoint: one more rounding equals the fp32 division (DESIGN R17)
    s_a = round_to_format(amax / 127.0, FP32)
    a32 = Az.astype(np.float32)
    s32 = s_a.astype(np.float32)
    with np.errstate(divide="ignore", invalid="ignore"):
        y = np.where(s32[:, None] > 0, a32 / np.where(s32 > 0, s32, np.float32(1))[:, None], np.float32(0))
    a_q = np.clip(round_half_away(y.astype(np.float64)), -127, 127).astype(np.int8)
    return ActQuant(a_q=a_q, s_a=s_a, status=0 if fin.all() else 1, rowsum=a_q.astype(np.int64).sum(axis=1))


@dataclass
class IntScaleQuant:
    q: np.ndarray          # int8 [N, K] codes in [-2^(b-1), 2^(b-1)-1]
    z: np.ndarray          # uint8 [G, N] integer group scales in [1, Z]
    sigma: np.ndarray      # float64 [N] per-column scales (fp32 values)
    status: int            # 0 ok; 1 non-finite input (column gets sigma 0, codes 0)


def quantize_intscale(W: np.ndarray, bits: int, group: int, Z: int = INTSCALE_Z) -> IntScaleQuant:
    """Group-wise linear absmax quantization with integer group scales (R15/R16), W[N, K]."""
    W = np.asarray(W, dtype=np.float64)
    N, K = W.shape
    if bits != 4:
        raise ValueError("integer group scales are defined for int4 weights (|q z| <= 128)")
    if group <= 0 or K % group:
        raise ValueError("group must divide K")
    G = K // group
    qmax = (1 << bits) - 1                                  # 2^b - 1 (App. A denominator)
    fin = np.isfinite(W).all(axis=1)                         # [N]
    Wz = np.where(fin[:, None], W, 0.0)
    amax = group_amax(Wz, group)                             # [G, N], exact
    amax_col = amax.max(axis=0)                              # [N]
    # 2 amax / (15 * 16) = amax / 120: periodic expansion (1/15), never an fp32 midpoint (R16)
    sigma = round_to_format(2.0 * amax_col / float(qmax * Z), FP32)
    sigma = np.where(fin, sigma, 0.0)                        # non-finite column: sigma 0, codes 0 (R5)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(sigma > 0, (2.0 * amax) / (float(qmax) * np.where(sigma > 0, sigma, 1.0)), 0.0)
    z = np.clip(np.ceil(ratio), 1, Z).astype(np.int64)      # [G, N]
    S = sigma[None, :] * z                                   # effective group scale, exact in float64
    S_full = np.repeat(S.T, group, axis=1)                   # [N, K]
    with np.errstate(divide="ignore", invalid="ignore"):
        y = np.where(S_full > 0, Wz / np.where(S_full > 0, S_full, 1.0), 0.0)
    lo, hi = -(1 << (bits - 1)), (1 << (bits - 1)) - 1
    q = np.clip(round_half_away(y), lo, hi).astype(np.int8)
    return IntScaleQuant(q=q, z=z.astype(np.uint8), sigma=sigma, status=0 if fin.all() else 1)


def gemm_i8(a_q: np.ndarray, s_a: np.ndarray, q: np.ndarray, z: np.ndarray, sigma: np.ndarray, group: int,
            cols=None):
    """acc[m, n] = sum_k a_q[m,k] * q[n,k] * z[k//g, n] as an exact integer (int64), then
    C[m, n] = acc * s_a[m] * sigma[n] in float64 and D[m, n] = sum_k |same terms| * s_a * sigma.
    Returns (C, D, acc)."""
    a = np.asarray(a_q, dtype=np.int64)
    q = np.asarray(q, dtype=np.int64)
    z = np.asarray(z, dtype=np.int64)
    sigma = np.asarray(sigma, dtype=np.float64)
    if cols is not None:
        cols = np.asarray(cols)
        q, z, sigma = q[cols], z[:, cols], sigma[cols]
    wz = q * np.repeat(z.T, group, axis=1)                   # [n, K] integers q * z
    acc = a @ wz.T                                           # exact int64
    dabs = np.abs(a) @ np.abs(wz).T
    sc = np.asarray(s_a, dtype=np.float64)[:, None] * sigma[None, :]
    return acc.astype(np.float64) * sc, dabs.astype(np.float64) * sc, acc
