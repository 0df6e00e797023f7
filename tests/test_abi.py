"""CPU-only checks of the C-ABI library: it loads, exports every symbol fq.h declares, and its
host-side logic (sizes, ladder, decision, validation) behaves as documented.  No compute calls."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "fq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fq_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def fq():
    from paper_2308_09723_b200 import fq as m
    return m


def test_library_exports_every_declared_symbol(fq):
    lib = ctypes.CDLL(fq.LIB_PATH)
    names = header_functions()
    assert len(names) >= 13
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(fq.EXPORTED)


def test_sizes_and_ladder(fq):
    assert fq.fq_codes_bytes(12288, 49152, 4) == 12288 * 49152 // 2
    assert fq.fq_codes_bytes(12288, 49152, 8) == 12288 * 49152
    assert fq.fq_codes_bytes(12288, 49152, 3) == 12288 * 49152 * 3 // 8   # int3 bit stream (R19)
    assert fq.fq_codes_bytes(12288, 49152, 2) == 12288 * 49152 // 4
    assert fq.fq_codes_bytes(12288, 49152, 5) == 0
    assert fq.fq_scales_bytes(12288, 49152, 128, fq.FQ_BF16) == 96 * 49152 * 2
    assert fq.fq_scales_bytes(12288, 49152, 100, fq.FQ_BF16) == 0
    from oracle import fq_oracle as O
    for K in (128, 4096, 12288, 49152, 7168, 96):
        lad = O.adapt_ladder(K, 16)
        assert fq.fq_adapt_levels(K, 16) == len(lad)
        assert [fq.fq_adapt_group_at(K, 16, L) for L in range(len(lad))] == lad
    assert fq.fq_adapt_decide(12288, 16, [1, 1, 0, 1]) == 3072
    assert fq.fq_adapt_decide(12288, 16, [0, 1]) == 12288
    assert fq.fq_adapt_decide(4096, 16, [1] * 8) == 16


def test_decide_matches_oracle_decide(fq):
    from oracle import fq_oracle as O
    import itertools
    for flags in itertools.product([0, 1], repeat=4):
        assert fq.fq_adapt_decide(4096, 256, list(flags)) == O.adapt_decide([bool(f) for f in flags], 4096, 256)


def test_validation_is_synchronous_and_launch_free(fq):
    """Invalid descriptors are rejected before any device work (pointers are dummies)."""
    dummy = ctypes.c_void_p(16)
    for bits in (5, 6, 7, 1):  # no kernel
        d = fq.make_wdesc(256, 256, bits, 64, fq.FQ_BF16)
        st = fq._lib.fq_gemm(dummy, fq.FQ_BF16, 1, ctypes.byref(d), dummy, dummy, dummy, fq.FQ_BF16,
                             None, 0, None)
        assert st == fq.FQ_ERR_UNSUPPORTED
    # int3 / int2: decode kernel only -- K % 128, and M beyond the decode kernel is refused
    d3 = fq.make_wdesc(192, 256, 3, 64, fq.FQ_BF16)
    assert fq._lib.fq_quantize(dummy, 0, ctypes.byref(d3), dummy, dummy, None, None) == fq.FQ_ERR_SHAPE
    d3 = fq.make_wdesc(256, 256, 3, 64, fq.FQ_BF16)
    assert fq._lib.fq_gemm(dummy, 0, 17, ctypes.byref(d3), dummy, dummy, dummy, 0, None, 0,
                           None) == fq.FQ_ERR_UNSUPPORTED  # per-element-scale path: M <= 16
    d2 = fq.make_wdesc(256, 256, 2, 128, fq.FQ_BF16)
    assert fq._lib.fq_gemm(dummy, 0, 33, ctypes.byref(d2), dummy, dummy, dummy, 0, None, 0,
                           None) == fq.FQ_ERR_UNSUPPORTED  # nibble path: M <= 32
    assert fq.fq_gemm_workspace_bytes(64, d2) == 0
    for bad in (fq.make_wdesc(250, 256, 4, 64, 0), fq.make_wdesc(256, 252, 4, 64, 0),
                fq.make_wdesc(256, 256, 4, 48, 0), fq.make_wdesc(256, 256, 4, 24, 0)):
        assert fq._lib.fq_quantize(dummy, 0, ctypes.byref(bad), dummy, dummy, None, None) == fq.FQ_ERR_SHAPE
    d = fq.make_wdesc(256, 256, 4, 64, fq.FQ_BF16)
    assert fq._lib.fq_gemm(dummy, fq.FQ_FP16, 1, ctypes.byref(d), dummy, dummy, dummy, fq.FQ_FP16,
                           None, 0, None) == fq.FQ_ERR_UNSUPPORTED  # scale dtype != activation dtype
    assert fq._lib.fq_gemm(None, 0, 1, ctypes.byref(d), dummy, dummy, dummy, 0, None, 0, None) == fq.FQ_ERR_INVALID_ARG
    assert fq._lib.fq_adapt_flags(dummy, 0, 256, 8, 0, 16, dummy, None, None) == fq.FQ_ERR_INVALID_ARG
    assert fq._lib.fq_adapt_flags(dummy, 0, 256, 8, 1001, 16, dummy, None, None) == fq.FQ_ERR_INVALID_ARG
    assert fq.fq_status_str(fq.FQ_ERR_SHAPE) == "FQ_ERR_SHAPE"
    # long columns are quantized in K-slices: only a group longer than one CTA can hold is refused
    per_col = fq.make_wdesc(131072, 256, 4, 131072, fq.FQ_BF16)
    assert fq._lib.fq_quantize(dummy, 0, ctypes.byref(per_col), dummy, dummy, None, None) == fq.FQ_ERR_SHAPE
    g32k = fq.make_wdesc(65536, 256, 4, 65536, fq.FQ_BF16)
    assert fq._lib.fq_quantize(dummy, fq.FQ_FP32, ctypes.byref(g32k), dummy, dummy, None, None) == fq.FQ_ERR_SHAPE
    # W and codes feed 16-byte loads / bulk copies: misaligned pointers are refused before any launch
    odd = ctypes.c_void_p(16 + 8)
    assert fq._lib.fq_quantize(odd, 0, ctypes.byref(d), dummy, dummy, None, None) == fq.FQ_ERR_INVALID_ARG
    assert fq._lib.fq_quantize(dummy, 0, ctypes.byref(d), odd, dummy, None, None) == fq.FQ_ERR_INVALID_ARG
    assert fq._lib.fq_quantize_rowshard(odd, 0, ctypes.byref(d), 2, 0, None, dummy, dummy, None,
                                        None) == fq.FQ_ERR_INVALID_ARG


def test_empty_batches_are_launch_free_noops(fq):
    """M == 0 (fq_gemm) and T == 0 / empty experts (fq_gemm_grouped) validate their arguments and
    return FQ_OK without touching the device (dummy pointers, no GPU needed)."""
    dummy = ctypes.c_void_p(16)
    d = fq.make_wdesc(4096, 16384, 4, 128, fq.FQ_BF16)
    assert fq._lib.fq_gemm(dummy, fq.FQ_BF16, 0, ctypes.byref(d), dummy, dummy, dummy, fq.FQ_BF16,
                           None, 0, None) == fq.FQ_OK
    assert fq._lib.fq_gemm(None, fq.FQ_BF16, 0, ctypes.byref(d), dummy, dummy, None, fq.FQ_BF16,
                           None, 0, None) == fq.FQ_OK  # zero-size A / C buffers may be NULL
    assert fq._lib.fq_gemm(dummy, fq.FQ_BF16, -1, ctypes.byref(d), dummy, dummy, dummy, fq.FQ_BF16,
                           None, 0, None) == fq.FQ_ERR_SHAPE
    bad = fq.make_wdesc(4096, 16384, 4, 96, fq.FQ_BF16)  # the empty batch still validates the descriptor
    assert fq._lib.fq_gemm(dummy, fq.FQ_BF16, 0, ctypes.byref(bad), dummy, dummy, dummy, fq.FQ_BF16,
                           None, 0, None) == fq.FQ_ERR_SHAPE
    E = 4
    offs = (ctypes.c_int64 * (E + 1))(*([0] * (E + 1)))
    groups = (ctypes.c_int32 * E)(*([128] * E))
    ptrs = (ctypes.c_void_p * E)(*([16] * E))
    assert fq._lib.fq_gemm_grouped(dummy, fq.FQ_BF16, 0, offs, E, ctypes.byref(d), groups, ptrs, ptrs, dummy,
                                   fq.FQ_BF16, None, 0, None) == fq.FQ_OK
    assert fq._lib.fq_gemm_grouped(None, fq.FQ_BF16, 0, offs, E, ctypes.byref(d), groups, ptrs, ptrs, None,
                                   fq.FQ_BF16, None, 0, None) == fq.FQ_OK


def test_gemm_workspace_sizes(fq):
    """Workspace contract (fq.h): 64 KiB counter region first; decode paths add partials + the
    pre-converted activations; the tensor-core path adds split-K partials only when its output
    tiles cannot fill the GPU.  Pure host logic (no device calls)."""
    d = fq.make_wdesc(12288, 49152, 4, 128, fq.FQ_BF16)
    for M in (1, 8, 16):  # decode path
        assert fq.fq_gemm_workspace_bytes(M, d) >= 65536 + M * 12288 * 2
    # 17..32 tokens: the tensor-core path by default (384 tiles, no split), the decode kernel's
    # four-token-tile class when forced
    assert fq.fq_gemm_workspace_bytes(32, d) == 256
    assert fq.fq_gemm_workspace_bytes_ex(32, d, fq.make_opts("decode")) >= 65536 + 32 * 12288 * 2
    big = fq.make_wdesc(12288, 49152, 4, 128, fq.FQ_BF16)
    assert fq.fq_gemm_workspace_bytes(2048, big) == 256           # 384 x 8 tiles fill the GPU: no split
    small = fq.make_wdesc(4096, 512, 4, 128, fq.FQ_BF16)
    nb = fq.fq_gemm_workspace_bytes(64, small)                    # 4 tiles: split-K partials
    assert nb > 65536 and (nb - 65536) % (4 * 64 * 128 * 4) == 0
    g64 = fq.make_wdesc(5120, 5120, 4, 64, fq.FQ_FP16)
    assert fq.fq_gemm_workspace_bytes(16, g64) >= 65536 + 16 * 5120 * 2  # group-split nibble path
    assert fq.fq_gemm_workspace_bytes(0, d) == 0
    assert fq.fq_gemm_grouped_workspace_bytes(64 * 16, 64, fq.make_wdesc(4096, 16384, 4, 4096, 0)) >= 65536
    # OPT-175B FC2 (K = 49152, N = 12288): 96 one-half tiles leave SMs idle -> two-half (256-row)
    # tiles with split-K partials [items][bn][256]; 17..32 tokens route to the same tensor-core path
    fc2 = fq.make_wdesc(49152, 12288, 4, 128, fq.FQ_BF16)
    nb = fq.fq_gemm_workspace_bytes(64, fc2)
    assert nb > 65536 and (nb - 65536) % (64 * 256 * 4) == 0
    forced = fq.fq_gemm_workspace_bytes_ex(32, fc2, fq.make_opts("tc"))
    dec = fq.fq_gemm_workspace_bytes_ex(32, fc2, fq.make_opts("decode"))
    assert forced != dec and fq.fq_gemm_workspace_bytes(32, fc2) == forced
    assert fq.fq_gemm_workspace_bytes_ex(32, fc2, None) == forced
    # ... and so does FC1 (384 one-half tiles, two CTAs per SM: no split, no partials)
    assert fq.fq_gemm_workspace_bytes(32, d) == fq.fq_gemm_workspace_bytes_ex(32, d, fq.make_opts("tc")) == 256


def test_routing_is_environment_independent(fq, monkeypatch):
    """fq.h: routing and split plans read nothing from the process environment (round-1 diagnostic
    switches are gone from the product build); overrides go through fq_gemm_opts only."""
    fc2 = fq.make_wdesc(49152, 12288, 4, 128, fq.FQ_BF16)
    base = {M: fq.fq_gemm_workspace_bytes(M, fc2) for M in (1, 16, 32, 64, 2048)}
    for k, v in (("FQ_GEMM_PATH", "decode"), ("FQ_GEMV_SPLITS", "1"), ("FQ_TC_HM", "1"), ("FQ_TC_SPLITS", "1"),
                 ("FQ_DECODE_TC", "1"), ("FQ_PDL", "0")):
        monkeypatch.setenv(k, v)
    assert {M: fq.fq_gemm_workspace_bytes(M, fc2) for M in base} == base
    so = open(fq.LIB_PATH, "rb").read()
    for name in (b"FQ_GEMM_PATH", b"FQ_GEMV_SPLITS", b"FQ_TC_HM", b"FQ_DECODE_TC", b"FQ_DEC_DEBUG", b"FQ_PDL"):
        assert name not in so, name


def test_gemm_opts_validation(fq):
    dummy = ctypes.c_void_p(16)
    d = fq.make_wdesc(4096, 512, 4, 128, fq.FQ_BF16)
    for bad in (fq.make_opts(3), fq.make_opts(0, -1), fq.make_opts(0, 0, 3), fq.make_opts(0, 0, 0, 5)):
        assert fq._lib.fq_gemm_ex(dummy, 0, 4, ctypes.byref(d), dummy, dummy, dummy, 0, None, 0, None,
                                  ctypes.byref(bad)) == fq.FQ_ERR_INVALID_ARG
        assert fq._lib.fq_gemm_workspace_bytes_ex(4, ctypes.byref(d), ctypes.byref(bad)) == 0
    o = fq.make_opts()
    o.reserved[2] = 1
    assert fq._lib.fq_gemm_ex(dummy, 0, 4, ctypes.byref(d), dummy, dummy, dummy, 0, None, 0, None,
                              ctypes.byref(o)) == fq.FQ_ERR_INVALID_ARG
    # decode split plans follow the override; A6 sizes follow tc_halves / splits
    s1 = fq.fq_gemm_workspace_bytes_ex(4, d, fq.make_opts("decode", 1))
    s4 = fq.fq_gemm_workspace_bytes_ex(4, d, fq.make_opts("decode", 4))
    assert s4 - s1 >= 4 * 4 * 512 * 4 - 256
    t1 = fq.fq_gemm_workspace_bytes_ex(64, d, fq.make_opts("tc", 1))
    t2 = fq.fq_gemm_workspace_bytes_ex(64, d, fq.make_opts("tc", 0, 2))
    assert t1 == 256 and t2 > 65536


def test_grouped_workspace_error_launches_nothing(fq):
    """fq.h: a call that returns != FQ_OK has written nothing -- the grouped call checks the
    workspace of every expert class before its first launch (dummy pointers: any launch would
    fault or return FQ_ERR_CUDA, and no GPU is needed to reach the check)."""
    dummy = ctypes.c_void_p(16)
    E = 3
    d = fq.make_wdesc(4096, 16384, 4, 128, fq.FQ_BF16)
    offs = (ctypes.c_int64 * (E + 1))(0, 100, 102, 110)   # one tensor-core expert, two decode experts
    groups = (ctypes.c_int32 * E)(128, 128, 16)
    ptrs = (ctypes.c_void_p * E)(16, 16, 16)
    assert fq._lib.fq_gemm_grouped(dummy, fq.FQ_BF16, 110, offs, E, ctypes.byref(d), groups, ptrs, ptrs, dummy,
                                   fq.FQ_BF16, dummy, 1024, None) == fq.FQ_ERR_WORKSPACE


def test_rowshard_validation(fq):
    dummy = ctypes.c_void_p(16)
    L = fq._lib
    # world must be a power of two whose K-slices sit on the ladder
    assert L.fq_adapt_flags_rowshard(dummy, 0, 12288, 256, 3, 0, 500, 16, dummy, dummy, None, None) == fq.FQ_ERR_SHAPE
    assert L.fq_adapt_flags_rowshard(dummy, 0, 12288, 256, 2, 2, 500, 16, dummy, dummy, None, None) == fq.FQ_ERR_INVALID_ARG
    assert L.fq_adapt_flags_rowshard(dummy, 0, 96, 256, 4, 0, 500, 16, dummy, dummy, None, None) == fq.FQ_ERR_SHAPE
    assert L.fq_adapt_flags_rowshard(dummy, 0, 12288, 256, 2, 0, 500, 16, dummy, None, None, None) == fq.FQ_ERR_INVALID_ARG
    assert L.fq_adapt_flags_cross(dummy, 12288, 256, 1, 500, 16, dummy, None) == fq.FQ_OK  # nothing spans shards
    d = fq.make_wdesc(12288, 256, 4, 12288, fq.FQ_BF16)
    # group > K/world needs the column-max table
    assert L.fq_quantize_rowshard(dummy, 0, ctypes.byref(d), 4, 0, None, dummy, dummy, None, None) == fq.FQ_ERR_INVALID_ARG
    d = fq.make_wdesc(12288, 256, 4, 96 * 16, fq.FQ_BF16)  # 1536 does not nest with 12288/16 = 768?  it does
    assert L.fq_quantize_rowshard(dummy, 0, ctypes.byref(d), 3, 0, None, dummy, dummy, None, None) == fq.FQ_ERR_INVALID_ARG


def test_i8_path_sizes_and_validation(fq):
    """int8-activation path (NEXT-4): sizes and shape / argument validation before any launch."""
    assert fq.fq_zscales_bytes(12288, 49152, 128) == 96 * 49152
    assert fq.fq_zscales_bytes(12288, 49152, 48) == 0      # group % 32
    assert fq.fq_zscales_bytes(12288, 49152, 96) == 0      # neither divides nor is a multiple of 128
    assert fq.fq_zscales_bytes(12288, 49152, 384) == 96 * 49152 // 3
    assert fq.fq_zscales_bytes(12300, 49152, 32) == 0      # K % 128
    assert fq.fq_zscales_bytes(12288, 49160, 128) == 0     # N % 16
    assert fq.fq_zscales_bytes(131072, 256, 128) == 0      # K > 65536 (int32 accumulator bound)
    assert fq.fq_gemm_i8_workspace_bytes(0, 1024, 256) == 0
    dummy = ctypes.c_void_p(16)
    L = fq._lib
    assert L.fq_gemm_i8(dummy, dummy, dummy, 4, 1024, 250, 128, dummy, dummy, dummy, dummy, fq.FQ_BF16, None, 0,
                        None) == fq.FQ_ERR_SHAPE
    assert L.fq_gemm_i8(dummy, dummy, dummy, 4, 1024, 256, 96, dummy, dummy, dummy, dummy, fq.FQ_BF16, None, 0,
                        None) == fq.FQ_ERR_SHAPE
    assert L.fq_gemm_i8(dummy, dummy, dummy, 4, 1024, 256, 128, None, dummy, dummy, dummy, fq.FQ_BF16, None, 0,
                        None) == fq.FQ_ERR_INVALID_ARG
    assert L.fq_gemm_i8(dummy, dummy, dummy, 4, 1024, 256, 128, dummy, dummy, dummy, dummy, 7, None, 0,
                        None) == fq.FQ_ERR_INVALID_ARG
    # empty batch: validated, nothing launched (A and C may be NULL)
    assert L.fq_gemm_i8(None, None, None, 0, 1024, 256, 128, dummy, dummy, dummy, None, fq.FQ_BF16, None, 0,
                        None) == fq.FQ_OK
    assert L.fq_quantize_acts_i8(dummy, fq.FQ_BF16, 2, 100, dummy, dummy, dummy, None, None) == fq.FQ_ERR_SHAPE
    assert L.fq_quantize_acts_i8(None, fq.FQ_BF16, 0, 128, None, None, None, None, None) == fq.FQ_OK
    assert L.fq_quantize_intscale(dummy, fq.FQ_BF16, 1024, 256, 48, dummy, dummy, dummy, None,
                                  None) == fq.FQ_ERR_SHAPE
    assert L.fq_quantize_intscale(dummy, 9, 1024, 256, 64, dummy, dummy, dummy, None,
                                  None) == fq.FQ_ERR_INVALID_ARG


def test_xr_sizes_and_validation(fq):
    """Fused row-parallel all-reduce (NEXT-1): buffer sizes follow the decode plan (256-column tiles x
    token tiles of 8 / 16 / 32), prefill-sized M and bad peer tables are refused before any launch."""
    d = fq.make_wdesc(6144, 12288, 4, 128, fq.FQ_BF16)   # an OPT-175B FC2 shard at t = 8
    for M, mt in ((1, 1), (8, 1), (16, 2), (32, 4)):
        tiles = (12288 // 256) * 1
        assert fq.fq_xr_counter_bytes(M, d) == tiles * 4
        assert fq.fq_xr_recv_bytes(M, d, 8) == tiles * 8 * (mt * 8 * 256) * 4
    assert fq.fq_xr_recv_bytes(33, d, 8) == 0 and fq.fq_xr_counter_bytes(64, d) == 0
    assert fq.fq_xr_recv_bytes(8, d, 0) == 0 and fq.fq_xr_recv_bytes(8, d, 9) == 0
    dummy = ctypes.c_void_p(16)
    pt = fq.fq_xr_peers()
    pt.world, pt.rank = 2, 0
    pt.recv[0] = pt.arrive[0] = pt.done[0] = pt.out[0] = 16   # rank 1's entries missing
    st = fq._lib.fq_gemm_allreduce(dummy, 0, 4, ctypes.byref(d), dummy, dummy, 0, ctypes.byref(pt), dummy,
                                   None, 0, None)
    assert st == fq.FQ_ERR_INVALID_ARG
    pt.recv[1] = pt.arrive[1] = pt.done[1] = pt.out[1] = 32
    st = fq._lib.fq_gemm_allreduce(dummy, 0, 40, ctypes.byref(d), dummy, dummy, 0, ctypes.byref(pt), dummy,
                                   None, 0, None)
    assert st == fq.FQ_ERR_UNSUPPORTED                    # M beyond the decode kernel


def test_grouped_dev_validation(fq):
    """fq_gemm_grouped_dev (device expert offsets): argument checks before any launch;
    T == 0 or a zero token bound launches nothing."""
    d = fq.make_wdesc(256, 256, 4, 64, fq.FQ_BF16)
    L = fq._lib
    E = 2
    grps = (ctypes.c_int32 * E)(64, 64)
    ptrs = (ctypes.c_void_p * E)(16, 16)
    dummy = ctypes.c_void_p(16)
    ws = ctypes.c_void_p(16)
    assert L.fq_gemm_grouped_dev(dummy, 0, 8, None, E, ctypes.byref(d), grps, ptrs, ptrs, dummy, 0, 8, None, ws,
                                 1 << 30, None) == fq.FQ_ERR_INVALID_ARG          # offsets missing
    bad = (ctypes.c_int32 * E)(64, 48)
    assert L.fq_gemm_grouped_dev(dummy, 0, 8, dummy, E, ctypes.byref(d), bad, ptrs, ptrs, dummy, 0, 8, None, ws,
                                 1 << 30, None) == fq.FQ_ERR_SHAPE                # an expert's group
    assert L.fq_gemm_grouped_dev(dummy, 0, 8, dummy, E, ctypes.byref(d), grps, ptrs, ptrs, dummy, 0, 8, None, None,
                                 0, None) == fq.FQ_ERR_WORKSPACE                  # decode experts need ws
    assert L.fq_gemm_grouped_dev(None, 0, 0, dummy, E, ctypes.byref(d), grps, ptrs, ptrs, None, 0, 8, None, None,
                                 0, None) == fq.FQ_OK                             # T == 0: nothing launched
    d3 = fq.make_wdesc(256, 256, 3, 64, fq.FQ_BF16)
    assert L.fq_gemm_grouped_dev(dummy, 0, 8, dummy, E, ctypes.byref(d3), grps, ptrs, ptrs, dummy, 0, 8, None, ws,
                                 1 << 30, None) == fq.FQ_ERR_UNSUPPORTED
