"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel (share of the step).
usage: python tools/launch_summary.py launches.csv 'header line'"""
import collections, csv, sys
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[1:]:
    if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]].replace(",", ""))
    if r[ix["Metric Unit"]] in ("nsecond", "ns"): v /= 1e3
    elif r[ix["Metric Unit"]] in ("msecond", "ms"): v *= 1e3
    k = r[ix["Kernel Name"]]
    tot[k] += v; cnt[k] += 1
T = sum(tot.values())
if len(sys.argv) > 2: print(sys.argv[2])
print(f"{'kernel':72s} launches   total us  share  mean us")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k[:72]:72s} {cnt[k]:8d} {v:10.1f} {v/T*100:5.1f}% {v/cnt[k]:8.2f}")
print(f"{'total':72s} {sum(cnt.values()):8d} {T:10.1f}")
