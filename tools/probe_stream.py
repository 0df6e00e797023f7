"""HBM streaming probes (diagnostics): read-only LDG sweep and the decode kernel's TMA access
pattern with no compute, over several box shapes / ring depths / CTAs per SM.
Usage (GPU box): python tools/probe_stream.py"""
import ctypes, itertools, os, subprocess, sys
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libprobe_stream.so")
if not os.path.exists(SO):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                           "-fPIC", "-o", SO, os.path.join(HERE, "probe_stream.cu")])
L = ctypes.CDLL(SO)
L.probe_ldg.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
L.probe_tma_setup.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 7
L.probe_tma_run.argtypes = [ctypes.c_int, ctypes.c_void_p]


def bench(fn, reps=40):
    for _ in range(5): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


def main():
    st = torch.cuda.current_stream().cuda_stream
    out = torch.zeros(4, dtype=torch.int32, device="cuda")
    big = torch.randint(0, 255, (2 * 1024**3,), dtype=torch.uint8, device="cuda")
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    for nbytes in (302 * 2**20, 1024 * 2**20, 2 * 1024**3):
        for grid_mul, block in ((1, 1024), (2, 1024), (4, 512), (8, 256), (16, 256)):
            us = bench(lambda: L.probe_ldg(big.data_ptr(), nbytes, nsm * grid_mul, block, out.data_ptr(), st))
            print(f"ldg {nbytes/2**20:6.0f} MiB grid={nsm*grid_mul} block={block}: {us:8.1f} us {nbytes/us/1e6:5.2f} TB/s", flush=True)
    del big

    for name, rows, rowbytes in (("FC1", 49152, 6144), ("FC2", 12288, 24576)):
        W = torch.randint(0, 255, (rows, rowbytes), dtype=torch.uint8, device="cuda")
        nbytes = rows * rowbytes
        for (R, C, nb), S, cps in itertools.product(((256, 64, 1), (256, 128, 1), (128, 128, 1), (128, 256, 1),
                                                    (64, 256, 1), (256, 64, 2), (128, 128, 2), (256, 256, 1)),
                                                   (4, 8), (1, 2, 3)):
            stage = R * C * nb
            if S * stage + 1024 > 227 * 1024 // cps: continue
            gx = rows // R
            best = None
            for splits in (1, 2, 3, 4, 6, 8, 12, 16):
                if rowbytes // (C * nb) < splits: continue
                if L.probe_tma_setup(W.data_ptr(), rows, rowbytes, R, C, nb, S, splits) != 0:
                    print("setup failed", R, C, nb); break
                pad = (227 * 1024) // cps - 2048
                us = bench(lambda: L.probe_tma_run(pad, st))
                ctas = L.probe_tma_ctas()
                if best is None or us < best[0]: best = (us, splits, ctas)
            if best:
                us, sp, ctas = best
                print(f"tma {name} box={R}x{C}x{nb} S={S} cta/sm={cps} best splits={sp} ctas={ctas}: {us:7.1f} us "
                      f"{nbytes/us/1e6:5.2f} TB/s", flush=True)


if __name__ == "__main__":
    main()
