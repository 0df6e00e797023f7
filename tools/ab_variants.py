"""A/B timing of compile-time kernel variants (diagnostics): each variant is libfq built with extra
-D flags (build.build_variant -> _variants/, selected with FQ_LIB_PATH) and timed by a tool script
in its own process, interleaved over rounds so box drift hits every variant alike.

    python tools/ab_variants.py --variant base= --variant pf0=FQ_DEC_PF=0,FQ_DEC_NIB_MAXREG=96 \\
        --rounds 2 -- tools/dec_sweep.py --M 1 8 --paths decode_mma
"""
import argparse, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2308_09723_b200 import build as B

ap = argparse.ArgumentParser()
ap.add_argument("--variant", action="append", default=[])
ap.add_argument("--rounds", type=int, default=1)
ap.add_argument("cmd", nargs=argparse.REMAINDER)
a = ap.parse_args()
cmd = a.cmd[1:] if a.cmd and a.cmd[0] == "--" else a.cmd
libs = {}
for v in a.variant:
    name, _, defs = v.partition("=")
    libs[name] = B.build_variant(name, [d for d in defs.split(",") if d])
for r in range(a.rounds):
    for name, lib in libs.items():
        env = dict(os.environ, FQ_LIB_PATH=lib)
        out = subprocess.run([sys.executable, os.path.join(ROOT, cmd[0])] + cmd[1:], env=env, capture_output=True,
                             text=True)
        for line in out.stdout.splitlines():
            print(f"r{r} {name:10s} {line}", flush=True)
        if out.returncode:
            print(name, out.stderr[-1500:], flush=True)
