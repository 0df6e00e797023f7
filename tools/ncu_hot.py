"""Per-instruction stall samples of an ncu report (SASS, address order), top-N windows.
usage: python tools/ncu_hot.py rep.ncu-rep [min_samples]"""
import csv, subprocess, sys
rep = sys.argv[1]; thr = int(sys.argv[2]) if len(sys.argv) > 2 else 20
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines())); hdr = rows[1]; data = rows[2:]; ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
def g(r, h):
    try: return int(r[ix[h]].replace(',', ''))
    except Exception: return 0
tot = sum(g(r, 'Warp Stall Sampling (All Samples)') for r in data)
for r in data:
    n = g(r, 'Warp Stall Sampling (All Samples)')
    if n >= thr:
        top = sorted(((g(r, h), h[6:]) for h in reasons), reverse=True)[:2]
        print(f"{r[ix['Address']][-5:]} {n:5d} {n/tot*100:4.1f}% {r[ix['Source']][:70]:70s} {top}")
