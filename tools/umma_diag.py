"""Diagnostics: build variants of the tcgen05 decode kernel with parts of the work removed
(FQ_DUMMA_DBG bits: 1 no MMA, 2 no tcgen05.st, 4 no tcgen05.ld, 8 no unpack) and time each on
OPT-175B FC1/FC2 int4 g128 in a subprocess (FQ_LIB_PATH selects the variant library)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2308_09723_b200 import build as B

variants = {"full": [], "noMMA": ["FQ_DUMMA_DBG=1"], "noSTTM": ["FQ_DUMMA_DBG=2"], "noLDTM": ["FQ_DUMMA_DBG=4"],
            "noUnpack": ["FQ_DUMMA_DBG=8"], "skeleton": ["FQ_DUMMA_DBG=15"]}
extra = sys.argv[1:]
for name, d in variants.items():
    lib = B.build_variant("umma_" + name, d + extra)
    env = dict(os.environ, FQ_LIB_PATH=lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "dec_sweep.py"), "--paths", "decode_umma",
                          "--M", "1", "16", "--reps", "20"], env=env, capture_output=True, text=True)
    for line in out.stdout.splitlines():
        print(f"{name:9s} {line}", flush=True)
    if out.returncode:
        print(name, out.stderr[-2000:])
