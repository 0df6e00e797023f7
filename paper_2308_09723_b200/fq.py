"""Thin Python binding of libfq.so (include/fq.h).  Argument marshalling only.

The `fq_*` functions mirror the C ABI one to one (same names, same arguments, torch tensors in
place of device pointers).  `quantize()` / `gemm()` / `gemm_grouped()` are the user-facing
conveniences built from them.  Every step of the hot path runs in the CUDA kernels of libfq.so;
there is no CPU or PyTorch fallback: if the library is missing or fails to load, importing this
module raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# FQ_LIB_PATH: diagnostics only (a variant built by build.build_variant, still in-tree)
LIB_PATH = os.environ.get("FQ_LIB_PATH") or os.path.join(_PKG, "libfq.so")

FQ_OK, FQ_ERR_INVALID_ARG, FQ_ERR_SHAPE, FQ_ERR_UNSUPPORTED, FQ_ERR_WORKSPACE, FQ_ERR_CUDA = range(6)
FQ_BF16, FQ_FP16, FQ_FP32 = 0, 1, 2
_DT = {torch.bfloat16: FQ_BF16, torch.float16: FQ_FP16, torch.float32: FQ_FP32}
_TD = {v: k for k, v in _DT.items()}


class FQError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {fq_status_str(status)}")


class fq_wdesc(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int64), ("N", ctypes.c_int64), ("bits", ctypes.c_int32),
                ("group", ctypes.c_int32), ("scale_dtype", ctypes.c_int32), ("reserved", ctypes.c_int32)]


FQ_PATH_AUTO, FQ_PATH_DECODE, FQ_PATH_TC = 0, 1, 2


class fq_gemm_opts(ctypes.Structure):
    """Routing / plan overrides (include/fq.h); all zero = the library's own plan."""
    _fields_ = [("path", ctypes.c_int32), ("splits", ctypes.c_int32), ("tc_halves", ctypes.c_int32),
                ("tc_dqg", ctypes.c_int32), ("reserved", ctypes.c_int32 * 4)]


def make_opts(path: str | int = 0, splits: int = 0, tc_halves: int = 0, tc_dqg: int = 0) -> fq_gemm_opts:
    if isinstance(path, str):
        path = {"auto": FQ_PATH_AUTO, "decode": FQ_PATH_DECODE, "tc": FQ_PATH_TC}[path]
    return fq_gemm_opts(path, splits, tc_halves, tc_dqg)


XR_MAX_WORLD = 8


class fq_xr_peers(ctypes.Structure):
    """Peer table of a fused row-parallel GEMM group (include/fq.h)."""
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("recv", ctypes.c_void_p * XR_MAX_WORLD), ("arrive", ctypes.c_void_p * XR_MAX_WORLD),
                ("done", ctypes.c_void_p * XR_MAX_WORLD), ("out", ctypes.c_void_p * XR_MAX_WORLD)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libfq.so not built ({LIB_PATH}); run __graft_entry__.build() "
                          "or python -m paper_2308_09723_b200.build")
    lib = ctypes.CDLL(LIB_PATH)
    c = ctypes
    P, I32, I64, U32, SZ = c.c_void_p, c.c_int32, c.c_int64, c.c_uint32, c.c_size_t
    WD = c.POINTER(fq_wdesc)
    sig = {
        "fq_version": (c.c_char_p, []),
        "fq_status_str": (c.c_char_p, [c.c_int]),
        "fq_codes_bytes": (SZ, [I64, I64, I32]),
        "fq_scales_bytes": (SZ, [I64, I64, I32, I32]),
        "fq_adapt_levels": (I32, [I64, I32]),
        "fq_adapt_group_at": (I32, [I64, I32, I32]),
        "fq_adapt_flags": (c.c_int, [P, I32, I64, I64, U32, I32, P, P, P]),
        "fq_adapt_decide": (I32, [I64, I32, c.POINTER(I32)]),
        "fq_adapt_flags_rowshard": (c.c_int, [P, I32, I64, I64, I32, I32, U32, I32, P, P, P, P]),
        "fq_adapt_flags_cross": (c.c_int, [P, I64, I64, I32, U32, I32, P, P]),
        "fq_quantize_rowshard": (c.c_int, [P, I32, WD, I32, I32, P, P, P, P, P]),
        "fq_quantize": (c.c_int, [P, I32, WD, P, P, P, P]),
        "fq_gemm_workspace_bytes": (SZ, [I64, WD]),
        "fq_gemm": (c.c_int, [P, I32, I64, WD, P, P, P, I32, P, SZ, P]),
        "fq_gemm_workspace_bytes_ex": (SZ, [I64, WD, c.POINTER(fq_gemm_opts)]),
        "fq_gemm_ex": (c.c_int, [P, I32, I64, WD, P, P, P, I32, P, SZ, P, c.POINTER(fq_gemm_opts)]),
        "fq_gemm_grouped_workspace_bytes": (SZ, [I64, I32, WD]),
        "fq_gemm_grouped": (c.c_int, [P, I32, I64, c.POINTER(I64), I32, WD, c.POINTER(I32),
                                      c.POINTER(P), c.POINTER(P), P, I32, P, SZ, P]),
        "fq_gemm_grouped_dev": (c.c_int, [P, I32, I64, P, I32, WD, c.POINTER(I32), c.POINTER(P), c.POINTER(P), P,
                                          I32, I64, P, P, SZ, P]),
        "fq_zscales_bytes": (SZ, [I64, I64, I32]),
        "fq_quantize_intscale": (c.c_int, [P, I32, I64, I64, I32, P, P, P, P, P]),
        "fq_quantize_acts_i8": (c.c_int, [P, I32, I64, I64, P, P, P, P, P]),
        "fq_gemm_i8_workspace_bytes": (SZ, [I64, I64, I64]),
        "fq_gemm_i8": (c.c_int, [P, P, P, I64, I64, I64, I32, P, P, P, P, I32, P, SZ, P]),
        "fq_xr_recv_bytes": (SZ, [I64, WD, I32]),
        "fq_xr_counter_bytes": (SZ, [I64, WD]),
        "fq_gemm_allreduce": (c.c_int, [P, I32, I64, WD, P, P, I32, c.POINTER(fq_xr_peers), P, P, SZ, P]),
        "fq_xr_wait": (c.c_int, [c.POINTER(fq_xr_peers), I64, WD, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


_lib = _load()
EXPORTED = ("fq_version", "fq_status_str", "fq_codes_bytes", "fq_scales_bytes", "fq_adapt_levels",
            "fq_adapt_group_at", "fq_adapt_flags", "fq_adapt_decide", "fq_adapt_flags_rowshard",
            "fq_adapt_flags_cross", "fq_quantize", "fq_quantize_rowshard", "fq_gemm_workspace_bytes",
            "fq_gemm", "fq_gemm_workspace_bytes_ex", "fq_gemm_ex", "fq_gemm_grouped_workspace_bytes",
            "fq_gemm_grouped", "fq_gemm_grouped_dev", "fq_zscales_bytes", "fq_quantize_intscale", "fq_quantize_acts_i8",
            "fq_gemm_i8_workspace_bytes", "fq_gemm_i8", "fq_xr_recv_bytes", "fq_xr_counter_bytes",
            "fq_gemm_allreduce", "fq_xr_wait")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(stream=None):
    if stream is not None:
        return ctypes.c_void_p(stream.cuda_stream)
    if _raw_stream is not None:  # the current stream's handle without building a Stream object
        return ctypes.c_void_p(_raw_stream(torch.cuda.current_device()))
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _check(st: int, what: str):
    if st != FQ_OK:
        raise FQError(st, what)


# ------------------------------------------------------------------------------ 1:1 ABI wrappers
def fq_version() -> str:
    return _lib.fq_version().decode()


def fq_status_str(s: int) -> str:
    return _lib.fq_status_str(s).decode()


def fq_codes_bytes(K: int, N: int, bits: int) -> int:
    return _lib.fq_codes_bytes(K, N, bits)


def fq_scales_bytes(K: int, N: int, group: int, scale_dtype: int) -> int:
    return _lib.fq_scales_bytes(K, N, group, scale_dtype)


def fq_adapt_levels(K: int, min_group: int) -> int:
    return _lib.fq_adapt_levels(K, min_group)


def fq_adapt_group_at(K: int, min_group: int, level: int) -> int:
    return _lib.fq_adapt_group_at(K, min_group, level)


def fq_adapt_flags(W: torch.Tensor, alpha_milli: int, min_group: int, flags: torch.Tensor,
                   status: torch.Tensor | None = None, stream=None) -> None:
    N, K = W.shape
    _check(_lib.fq_adapt_flags(_ptr(W), _DT[W.dtype], K, N, alpha_milli, min_group, _ptr(flags),
                               _ptr(status), _stream(stream)), "fq_adapt_flags")


def fq_adapt_decide(K: int, min_group: int, flags_host) -> int:
    arr = (ctypes.c_int32 * max(1, len(flags_host)))(*[int(f) for f in flags_host])
    return _lib.fq_adapt_decide(K, min_group, arr)


def fq_adapt_flags_rowshard(W_shard: torch.Tensor, K: int, world: int, rank: int, alpha_milli: int,
                            min_group: int, flags: torch.Tensor | None, colmax: torch.Tensor,
                            status: torch.Tensor | None = None, stream=None) -> None:
    N = W_shard.shape[0]
    _check(_lib.fq_adapt_flags_rowshard(_ptr(W_shard), _DT[W_shard.dtype], K, N, world, rank, alpha_milli,
                                        min_group, _ptr(flags), _ptr(colmax), _ptr(status), _stream(stream)),
           "fq_adapt_flags_rowshard")


def fq_adapt_flags_cross(colmax: torch.Tensor, K: int, N: int, world: int, alpha_milli: int, min_group: int,
                         flags: torch.Tensor, stream=None) -> None:
    _check(_lib.fq_adapt_flags_cross(_ptr(colmax), K, N, world, alpha_milli, min_group, _ptr(flags),
                                     _stream(stream)), "fq_adapt_flags_cross")


def fq_quantize_rowshard(W_shard: torch.Tensor, d: fq_wdesc, world: int, rank: int, colmax: torch.Tensor | None,
                         codes: torch.Tensor, scales: torch.Tensor, status: torch.Tensor | None = None,
                         stream=None) -> None:
    _check(_lib.fq_quantize_rowshard(_ptr(W_shard), _DT[W_shard.dtype], ctypes.byref(d), world, rank,
                                     _ptr(colmax), _ptr(codes), _ptr(scales), _ptr(status), _stream(stream)),
           "fq_quantize_rowshard")


def make_wdesc(K: int, N: int, bits: int, group: int, scale_dtype: int) -> fq_wdesc:
    return fq_wdesc(K, N, bits, group, scale_dtype, 0)


def fq_quantize(W: torch.Tensor, d: fq_wdesc, codes: torch.Tensor, scales: torch.Tensor,
                status: torch.Tensor | None = None, stream=None) -> None:
    _check(_lib.fq_quantize(_ptr(W), _DT[W.dtype], ctypes.byref(d), _ptr(codes), _ptr(scales),
                            _ptr(status), _stream(stream)), "fq_quantize")


def fq_gemm_workspace_bytes(M: int, d: fq_wdesc) -> int:
    return _lib.fq_gemm_workspace_bytes(M, ctypes.byref(d))


def fq_gemm(A: torch.Tensor, M: int, d: fq_wdesc, codes: torch.Tensor, scales: torch.Tensor,
            C: torch.Tensor, ws: torch.Tensor | None, stream=None) -> None:
    _check(_lib.fq_gemm(_ptr(A), _DT[A.dtype], M, ctypes.byref(d), _ptr(codes), _ptr(scales),
                        _ptr(C), _DT[C.dtype], _ptr(ws), 0 if ws is None else ws.numel() * ws.element_size(),
                        _stream(stream)), "fq_gemm")


def fq_gemm_workspace_bytes_ex(M: int, d: fq_wdesc, opts: fq_gemm_opts | None) -> int:
    return _lib.fq_gemm_workspace_bytes_ex(M, ctypes.byref(d), None if opts is None else ctypes.byref(opts))


def fq_gemm_ex(A: torch.Tensor, M: int, d: fq_wdesc, codes: torch.Tensor, scales: torch.Tensor,
               C: torch.Tensor, ws: torch.Tensor | None, stream=None, opts: fq_gemm_opts | None = None) -> None:
    _check(_lib.fq_gemm_ex(_ptr(A), _DT[A.dtype], M, ctypes.byref(d), _ptr(codes), _ptr(scales),
                           _ptr(C), _DT[C.dtype], _ptr(ws), 0 if ws is None else ws.numel() * ws.element_size(),
                           _stream(stream), None if opts is None else ctypes.byref(opts)), "fq_gemm_ex")


def fq_gemm_grouped_workspace_bytes(T: int, E: int, d: fq_wdesc) -> int:
    return _lib.fq_gemm_grouped_workspace_bytes(T, E, ctypes.byref(d))


def fq_gemm_grouped(A, T, offsets_host, E, d, groups_host, codes_ptrs, scales_ptrs, C, ws, stream=None):
    offs = (ctypes.c_int64 * (E + 1))(*[int(x) for x in offsets_host])
    grps = (ctypes.c_int32 * E)(*[int(x) for x in groups_host])
    cps = (ctypes.c_void_p * E)(*[int(x) for x in codes_ptrs])
    sps = (ctypes.c_void_p * E)(*[int(x) for x in scales_ptrs])
    _check(_lib.fq_gemm_grouped(_ptr(A), _DT[A.dtype], T, offs, E, ctypes.byref(d), grps, cps, sps,
                                _ptr(C), _DT[C.dtype], _ptr(ws),
                                0 if ws is None else ws.numel() * ws.element_size(), _stream(stream)),
           "fq_gemm_grouped")


def fq_gemm_grouped_dev(A, T, offsets_dev: torch.Tensor, E, d, groups_host, codes_ptrs, scales_ptrs, C, max_tokens,
                        ws, status: torch.Tensor | None = None, stream=None):
    grps = (ctypes.c_int32 * E)(*[int(x) for x in groups_host])
    cps = (ctypes.c_void_p * E)(*[int(x) for x in codes_ptrs])
    sps = (ctypes.c_void_p * E)(*[int(x) for x in scales_ptrs])
    _check(_lib.fq_gemm_grouped_dev(_ptr(A), _DT[A.dtype], T, _ptr(offsets_dev), E, ctypes.byref(d), grps, cps, sps,
                                    _ptr(C), _DT[C.dtype], max_tokens, _ptr(status), _ptr(ws),
                                    0 if ws is None else ws.numel() * ws.element_size(), _stream(stream)),
           "fq_gemm_grouped_dev")


def fq_zscales_bytes(K: int, N: int, group: int) -> int:
    return _lib.fq_zscales_bytes(K, N, group)


def fq_quantize_intscale(W: torch.Tensor, group: int, codes: torch.Tensor, zscales: torch.Tensor,
                         colscale: torch.Tensor, status: torch.Tensor | None = None, stream=None) -> None:
    N, K = W.shape
    _check(_lib.fq_quantize_intscale(_ptr(W), _DT[W.dtype], K, N, group, _ptr(codes), _ptr(zscales),
                                     _ptr(colscale), _ptr(status), _stream(stream)), "fq_quantize_intscale")


def fq_quantize_acts_i8(A: torch.Tensor, a_q: torch.Tensor, a_scale: torch.Tensor, a_rowsum: torch.Tensor,
                        status: torch.Tensor | None = None, stream=None) -> None:
    M, K = A.shape
    _check(_lib.fq_quantize_acts_i8(_ptr(A), _DT[A.dtype], M, K, _ptr(a_q), _ptr(a_scale), _ptr(a_rowsum),
                                    _ptr(status), _stream(stream)), "fq_quantize_acts_i8")


def fq_gemm_i8_workspace_bytes(M: int, K: int, N: int) -> int:
    return _lib.fq_gemm_i8_workspace_bytes(M, K, N)


def fq_gemm_i8(a_q: torch.Tensor, a_scale: torch.Tensor, a_rowsum: torch.Tensor, M: int, K: int, N: int,
               group: int, codes: torch.Tensor, zscales: torch.Tensor, colscale: torch.Tensor, C: torch.Tensor,
               ws: torch.Tensor | None, stream=None) -> None:
    _check(_lib.fq_gemm_i8(_ptr(a_q), _ptr(a_scale), _ptr(a_rowsum), M, K, N, group, _ptr(codes), _ptr(zscales), _ptr(colscale),
                           _ptr(C), _DT[C.dtype], _ptr(ws), 0 if ws is None else ws.numel() * ws.element_size(),
                           _stream(stream)), "fq_gemm_i8")


# ------------------------------------------------------------------------------ conveniences
_WS: dict = {}


def workspace(nbytes: int, device, stream=None) -> torch.Tensor:
    """Zero-filled scratch reused across calls (the kernels leave their counters zeroed).

    One buffer per (device, stream): calls sharing a workspace must be stream-ordered (fq.h), so
    calls on different streams get different buffers.  The buffer is allocated and zero-filled on
    the stream that uses it; a buffer replaced by a larger one is released to the caching allocator
    on that same stream, i.e. only after the kernels already enqueued there have finished."""
    dev = device if isinstance(device, torch.device) else torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    if stream is not None:
        h = stream.cuda_stream
    elif _raw_stream is not None:
        h = _raw_stream(idx)
    else:
        h = torch.cuda.current_stream(idx).cuda_stream
    key = (idx, h)
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        st = stream if stream is not None else torch.cuda.current_stream(idx)
        with torch.cuda.stream(st):
            ws = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device=torch.device("cuda", idx))
        _WS[key] = ws
    return ws


@dataclass
class QuantizedWeight:
    """Packed weights of one matrix in the canonical layout (include/fq.h)."""
    codes: torch.Tensor       # uint8 [N, K*bits/8]
    scales: torch.Tensor      # [K/group, N], activation dtype
    K: int
    N: int
    bits: int
    group: int

    @property
    def desc(self) -> fq_wdesc:
        return make_wdesc(self.K, self.N, self.bits, self.group, _DT[self.scales.dtype])

    @property
    def nbytes(self) -> int:
        return self.codes.numel() + self.scales.numel() * self.scales.element_size()


def adapt_group(W: torch.Tensor, alpha_milli: int = 500, min_group: int = 16, process_group=None) -> int:
    """Adaptive group size (§3.3): device flags (A1), optional OR across a process group
    (tensor-parallel shards of one matrix), host decision (A2)."""
    N, K = W.shape
    nlev = fq_adapt_levels(K, min_group)
    flags = torch.zeros(max(1, nlev - 1), dtype=torch.int32, device=W.device)
    fq_adapt_flags(W, alpha_milli, min_group, flags)
    if process_group is not None:
        import torch.distributed as dist
        dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=process_group)
    return fq_adapt_decide(K, min_group, flags.cpu().tolist()[: nlev - 1])


class _KernelOps:
    """The row-shard adaptive protocol's device steps (tp.rowshard_protocol) on the libfq kernels."""

    @staticmethod
    def alloc(nflags: int, world: int, N: int, device):
        # one int32 buffer [flags | colmax as fp32 bits]: non-negative fp32 values order like their
        # int32 bit patterns, so a single MAX all-reduce combines both
        buf = torch.zeros(nflags + world * N, dtype=torch.int32, device=device)
        return buf, buf[:nflags], buf[nflags:].view(torch.float32)

    @staticmethod
    def shard_pass(W_shard, K, world, rank, alpha_milli, min_group, flags, colmax):
        fq_adapt_flags_rowshard(W_shard, K, world, rank, alpha_milli, min_group,
                                flags if flags.numel() else None, colmax)

    @staticmethod
    def cross(colmax, K, N, world, alpha_milli, min_group, flags):
        if world > 1:
            fq_adapt_flags_cross(colmax, K, N, world, alpha_milli, min_group, flags)

    @staticmethod
    def decide(K, min_group, flags) -> int:
        return fq_adapt_decide(K, min_group, flags.cpu().tolist())


KERNEL_OPS = _KernelOps()


def quantize_rowshard(W_shard: torch.Tensor, K: int, world: int, rank: int, bits: int, group: int,
                      colmax: torch.Tensor | None = None, scale_dtype=torch.bfloat16,
                      status: torch.Tensor | None = None) -> QuantizedWeight:
    """Rank `rank`'s K-slice of the unsharded quantization of a row-parallel matrix (fq.h
    fq_quantize_rowshard): codes/scales are the K-/G-slices of fq_quantize(W_full, bits, group);
    `colmax` (the MAX-all-reduced [world, N] shard column maxima) is needed when group > K/world."""
    assert W_shard.is_cuda and W_shard.dim() == 2 and W_shard.is_contiguous()
    N, Ks = W_shard.shape
    assert Ks * world == K
    gs = min(group, Ks)
    d = make_wdesc(K, N, bits, group, _DT[scale_dtype])
    codes = torch.empty((N, Ks * bits // 8), dtype=torch.uint8, device=W_shard.device)
    scales = torch.empty((Ks // gs, N), dtype=scale_dtype, device=W_shard.device)
    fq_quantize_rowshard(W_shard, d, world, rank, colmax, codes, scales, status)
    return QuantizedWeight(codes, scales, Ks, N, bits, gs)


def quantize(W: torch.Tensor, bits: int = 4, group: int | None = 128, scale_dtype=torch.bfloat16,
             alpha_milli: int = 500, min_group: int = 16, status: torch.Tensor | None = None) -> QuantizedWeight:
    """fq_quantize(W, bits, group | adaptive): W is [N, K] (nn.Linear layout) on a CUDA device.
    group=None selects the adaptive group size."""
    assert W.is_cuda and W.dim() == 2 and W.is_contiguous()
    N, K = W.shape
    if group is None:
        group = adapt_group(W, alpha_milli, min_group)
    d = make_wdesc(K, N, bits, group, _DT[scale_dtype])
    codes = torch.empty((N, K * bits // 8), dtype=torch.uint8, device=W.device)
    scales = torch.empty((K // group, N), dtype=scale_dtype, device=W.device)
    fq_quantize(W, d, codes, scales, status)
    return QuantizedWeight(codes, scales, K, N, bits, group)


def gemm_grouped(A: torch.Tensor, offsets, experts: list, out: torch.Tensor | None = None,
                 out_dtype=None, stream=None) -> torch.Tensor:
    """MoE expert batch: rows offsets[e]:offsets[e+1] of A (sorted by expert) times expert e.
    All experts share K, N, bits and scale dtype; each has its own group size (adaptive)."""
    assert A.is_cuda and A.dim() == 2 and A.is_contiguous()
    E = len(experts)
    offs = [int(x) for x in offsets]
    assert len(offs) == E + 1
    q0 = experts[0]
    T = A.shape[0]
    if out is None:
        out = torch.empty((T, q0.N), dtype=out_dtype or A.dtype, device=A.device)
    d = q0.desc
    nb = fq_gemm_grouped_workspace_bytes(T, E, d)
    ws = workspace(nb, A.device, stream)
    fq_gemm_grouped(A, T, offs, E, d, [q.group for q in experts], [q.codes.data_ptr() for q in experts],
                    [q.scales.data_ptr() for q in experts], out, ws, stream)
    return out


def gemm_grouped_dev(A: torch.Tensor, offsets_dev: torch.Tensor, experts: list, max_tokens: int,
                     out: torch.Tensor | None = None, out_dtype=None, status: torch.Tensor | None = None,
                     stream=None) -> torch.Tensor:
    """MoE expert batch with the routing offsets on the device (int64 [E+1]): no host sync.
    `max_tokens` bounds every expert's token count (rows beyond it are not computed; status bit 2)."""
    assert A.is_cuda and A.dim() == 2 and A.is_contiguous()
    assert offsets_dev.is_cuda and offsets_dev.dtype == torch.int64 and offsets_dev.numel() == len(experts) + 1
    E = len(experts)
    q0 = experts[0]
    T = A.shape[0]
    if out is None:
        out = torch.empty((T, q0.N), dtype=out_dtype or A.dtype, device=A.device)
    d = q0.desc
    ws = workspace(fq_gemm_grouped_workspace_bytes(T, E, d), A.device, stream)
    fq_gemm_grouped_dev(A, T, offsets_dev, E, d, [q.group for q in experts], [q.codes.data_ptr() for q in experts],
                        [q.scales.data_ptr() for q in experts], out, max_tokens, ws, status, stream)
    return out


def gemm(A: torch.Tensor, qw: QuantizedWeight, out: torch.Tensor | None = None,
         out_dtype=None, stream=None, opts: fq_gemm_opts | None = None) -> torch.Tensor:
    """C[M, N] = A[M, K] . dequant(qw)^T  (fused, on the GPU).  `opts` (make_opts(...)) overrides
    the library's routing / split plan (tests, measurements)."""
    assert A.is_cuda and A.dim() == 2 and A.is_contiguous() and A.shape[1] == qw.K
    M = A.shape[0]
    d = qw.desc
    if out is None:
        out = torch.empty((M, qw.N), dtype=out_dtype or A.dtype, device=A.device)
    okey = None if opts is None else (opts.path, opts.splits, opts.tc_halves, opts.tc_dqg)
    key = (M, qw.K, qw.N, qw.bits, qw.group, okey)
    nb = _WS_BYTES.get(key)
    if nb is None:
        nb = _WS_BYTES[key] = fq_gemm_workspace_bytes_ex(M, d, opts)
    ws = workspace(nb, A.device, stream)
    if opts is None:
        fq_gemm(A, M, d, qw.codes, qw.scales, out, ws, stream)
    else:
        fq_gemm_ex(A, M, d, qw.codes, qw.scales, out, ws, stream, opts)
    return out


# (M, K, N, bits, group, opts) -> workspace bytes: a pure function of its key (fq.h: routing reads
# nothing but the arguments)
_WS_BYTES: dict = {}


# ------------------------------------------------------------------------------ int8-activation path
@dataclass
class QuantizedWeightI8:
    """int4 codes with integer group scales (fq.h fq_quantize_intscale)."""
    codes: torch.Tensor       # uint8 [N, K/2] canonical int4
    zscales: torch.Tensor     # uint8 [K/group, N], values 1..16
    colscale: torch.Tensor    # float32 [N]
    K: int
    N: int
    group: int

    @property
    def nbytes(self) -> int:
        return self.codes.numel() + self.zscales.numel() + self.colscale.numel() * 4


def quantize_intscale(W: torch.Tensor, group: int = 128, status: torch.Tensor | None = None) -> QuantizedWeightI8:
    assert W.is_cuda and W.dim() == 2 and W.is_contiguous()
    N, K = W.shape
    codes = torch.empty((N, K // 2), dtype=torch.uint8, device=W.device)
    z = torch.empty((K // group, N), dtype=torch.uint8, device=W.device)
    sg = torch.empty((N,), dtype=torch.float32, device=W.device)
    fq_quantize_intscale(W, group, codes, z, sg, status)
    return QuantizedWeightI8(codes, z, sg, K, N, group)


def quantize_acts_i8(A: torch.Tensor, status: torch.Tensor | None = None, stream=None):
    """Per-token int8 activations: returns (a_q int8 [M, K], a_scale float32 [M], a_rowsum int32 [M])."""
    assert A.is_cuda and A.dim() == 2 and A.is_contiguous()
    M, K = A.shape
    a_q = torch.empty((M, K), dtype=torch.int8, device=A.device)
    sa = torch.empty((M,), dtype=torch.float32, device=A.device)
    rs = torch.empty((M,), dtype=torch.int32, device=A.device)
    fq_quantize_acts_i8(A, a_q, sa, rs, status, stream)
    return a_q, sa, rs


def gemm_i8(A: torch.Tensor | None, qw: QuantizedWeightI8, out: torch.Tensor | None = None, out_dtype=None,
            stream=None, acts=None) -> torch.Tensor:
    """C[M, N] = s_a * sigma * (a_q . (q z)^T): quantizes A per token to int8 (unless `acts` =
    (a_q, a_scale, a_rowsum) is given), then the tcgen05 kind::i8 GEMM."""
    a_q, sa, rs = acts if acts is not None else quantize_acts_i8(A, stream=stream)
    M = a_q.shape[0]
    if out is None:
        out = torch.empty((M, qw.N), dtype=out_dtype or (A.dtype if A is not None else torch.bfloat16),
                          device=a_q.device)
    nb = fq_gemm_i8_workspace_bytes(M, qw.K, qw.N)
    ws = workspace(nb, a_q.device, stream)
    fq_gemm_i8(a_q, sa, rs, M, qw.K, qw.N, qw.group, qw.codes, qw.zscales, qw.colscale, out, ws, stream)
    return out


# ------------------------------------------------------------------------------ fused row-parallel all-reduce
def fq_xr_recv_bytes(M: int, d: fq_wdesc, world: int) -> int:
    return _lib.fq_xr_recv_bytes(M, ctypes.byref(d), world)


def fq_xr_counter_bytes(M: int, d: fq_wdesc) -> int:
    return _lib.fq_xr_counter_bytes(M, ctypes.byref(d))


def fq_gemm_allreduce(A: torch.Tensor, M: int, d: fq_wdesc, codes: torch.Tensor, scales: torch.Tensor, cdt: int,
                      peers: fq_xr_peers, peers_dev: torch.Tensor, ws: torch.Tensor | None, stream=None) -> None:
    _check(_lib.fq_gemm_allreduce(_ptr(A), _DT[A.dtype], M, ctypes.byref(d), _ptr(codes), _ptr(scales), cdt,
                                  ctypes.byref(peers), _ptr(peers_dev), _ptr(ws),
                                  0 if ws is None else ws.numel() * ws.element_size(), _stream(stream)),
           "fq_gemm_allreduce")


def fq_xr_wait(peers: fq_xr_peers, M: int, d: fq_wdesc, stream=None) -> None:
    _check(_lib.fq_xr_wait(ctypes.byref(peers), M, ctypes.byref(d), _stream(stream)), "fq_xr_wait")


class XRRank:
    """One rank's view of a fused row-parallel GEMM group: its peer table (host + device copy) and
    its output buffer.  Build with xr_group_local (all ranks on one device: tests, one-GPU
    diagnostics) or xr_group_symmetric (one rank per GPU, peer memory from torch symmetric memory)."""

    def __init__(self, peers: fq_xr_peers, out: torch.Tensor, keep: list):
        self.peers = peers
        self.out = out
        raw = bytes(peers)
        self.peers_dev = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(out.device)
        self._keep = keep  # the buffers the table points into

    def gemm(self, A: torch.Tensor, qw_shard: "QuantizedWeight", stream=None) -> torch.Tensor:
        """out = sum over ranks of A_r . dequant(W_r)^T, on every rank; stream-ordered (fq_xr_wait)."""
        M = A.shape[0]
        d = qw_shard.desc
        nb = fq_gemm_workspace_bytes_ex(M, d, make_opts("decode"))  # the decode kernel's plan
        ws = workspace(nb, A.device, stream)
        fq_gemm_allreduce(A, M, d, qw_shard.codes, qw_shard.scales, _DT[self.out.dtype], self.peers,
                          self.peers_dev, ws, stream)
        fq_xr_wait(self.peers, M, d, stream)
        return self.out


def gemv_max_m(bits: int, group: int) -> int:
    """Largest M the decode kernel serves in one pass (fq.h: 32 on the nibble path, else 16); the
    fused all-reduce GEMM needs M within it."""
    return 32 if bits <= 4 and group % 128 == 0 else 16


def _xr_sizes(M: int, d: fq_wdesc, world: int):
    rb, cb = fq_xr_recv_bytes(M, d, world), fq_xr_counter_bytes(M, d)
    if rb == 0 or cb == 0:
        raise FQError(FQ_ERR_UNSUPPORTED, "fused all-reduce: M beyond the decode kernel or bad shard")
    return rb, cb


def xr_group_local(world: int, M: int, d: fq_wdesc, out_dtype=torch.bfloat16, device="cuda") -> list:
    """Every rank of a group on ONE device (pointers are plain device addresses)."""
    assert 1 <= world <= XR_MAX_WORLD
    rb, cb = _xr_sizes(M, d, world)
    recv = [torch.zeros(rb // 4, dtype=torch.float32, device=device) for _ in range(world)]
    arrive = [torch.zeros(cb // 4, dtype=torch.int32, device=device) for _ in range(world)]
    done = [torch.zeros(1, dtype=torch.int32, device=device) for _ in range(world)]
    outs = [torch.zeros((M, d.N), dtype=out_dtype, device=device) for _ in range(world)]
    keep = recv + arrive + done + outs
    ranks = []
    for r in range(world):
        pt = fq_xr_peers()
        pt.world, pt.rank = world, r
        for q in range(world):
            pt.recv[q], pt.arrive[q] = recv[q].data_ptr(), arrive[q].data_ptr()
            pt.done[q], pt.out[q] = done[q].data_ptr(), outs[q].data_ptr()
        ranks.append(XRRank(pt, outs[r], keep))
    return ranks


def xr_group_symmetric(process_group, M: int, d: fq_wdesc, out_dtype=torch.bfloat16) -> XRRank:
    """This rank of a group with one rank per GPU: the receive slots, counters and outputs live in
    torch symmetric memory, whose peer mappings (NVLink) give every rank every other rank's address."""
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm
    world, rank = dist.get_world_size(process_group), dist.get_rank(process_group)
    assert 1 <= world <= XR_MAX_WORLD
    rb, cb = _xr_sizes(M, d, world)
    dev = torch.device("cuda", torch.cuda.current_device())
    ob = M * d.N * torch.tensor([], dtype=out_dtype).element_size()
    sizes = [rb, cb, 256, ob]
    offs = [0]
    for sz in sizes[:-1]:
        offs.append(offs[-1] + (sz + 255) // 256 * 256)
    try:
        symm.enable_symm_mem_for_group(process_group.group_name)
    except Exception:
        pass  # newer torch: implicit
    buf = symm.empty(offs[-1] + sizes[-1], dtype=torch.uint8, device=dev)
    buf.zero_()
    h = symm.rendezvous(buf, process_group)
    torch.cuda.synchronize()
    dist.barrier(group=process_group)
    pt = fq_xr_peers()
    pt.world, pt.rank = world, rank
    for q in range(world):
        base = int(h.buffer_ptrs[q])
        pt.recv[q], pt.arrive[q], pt.done[q], pt.out[q] = (base + o for o in offs)
    out = buf[offs[3]:offs[3] + ob].view(out_dtype).view(M, d.N)
    return XRRank(pt, out, [buf, h])
