"""Summarise an ncu report: top stall reasons (by opcode), instruction mix, key pipe metrics."""
import csv, collections, subprocess, sys
rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]; data = rows[2:]; ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot = collections.Counter(); byop = collections.defaultdict(collections.Counter); ninst = collections.Counter()
def g(r, h):
    try: return int(r[ix[h]].replace(',', ''))
    except Exception: return 0
for r in data:
    srcl = r[ix['Source']].strip()
    if not srcl: continue
    op = srcl.split()[0]
    if op.startswith('@'): op = srcl.split()[1]
    op = op.split('.')[0]
    ninst[op] += g(r, 'Instructions Executed')
    for h in reasons:
        tot[h] += g(r, h); byop[op][h] += g(r, h)
T = sum(tot.values())
print("samples", T, "instructions", sum(ninst.values()))
for h, v in tot.most_common(9):
    print(f"  {h:24s} {v/T*100:5.1f}%", collections.Counter({op: byop[op][h] for op in byop}).most_common(4))
print("mix", ninst.most_common(16))
top = sorted(data, key=lambda r: -g(r, 'Warp Stall Sampling (All Samples)'))[:10]
for r in top: print("  hot", r[ix['Address']][-5:], r[ix['Source']][:60], g(r, 'Warp Stall Sampling (All Samples)'))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines())); hdr = r[0]; vals = r[-1]
keys = ('gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__warps_eligible.avg.per_cycle_active', 'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread')
for h, v in zip(hdr, vals):
    if h in keys: print(f"  {h:70s} {v}")
