"""Per-instruction stall samples of one kernel's hottest loop from an ncu source-page CSV:
  ncu -i rep --page source --csv --kernel-name regex:NAME --print-source sass > k.csv
  python tools/sass_hot.py k.csv [min_exec] [max_exec]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
col = {h: i for i, h in enumerate(hdr)}
I = lambda r, h: int(r[col[h]] or 0)
ex = [I(r, 'Instructions Executed') for r in data]
lo = int(sys.argv[2]) if len(sys.argv) > 2 else max(ex) * 0.9
hi = int(sys.argv[3]) if len(sys.argv) > 3 else max(ex) * 1.1
tot = sum(I(r, 'Warp Stall Sampling (All Samples)') for r in data)
reasons = ['stall_math', 'stall_wait', 'stall_not_selected', 'stall_selected', 'stall_short_sb',
           'stall_dispatch', 'stall_barrier', 'stall_long_sb', 'stall_mio', 'stall_branch_resolving']
body = [r for r, e in zip(data, ex) if lo <= e <= hi]
s = sum(I(r, 'Warp Stall Sampling (All Samples)') for r in body)
print(f'{len(body)} instructions, {s} of {tot} samples ({s / max(tot, 1):.2f})')
agg = {k: sum(I(r, k) for r in body) for k in reasons}
print('  '.join(f'{k[6:]}={v}' for k, v in agg.items()))
print('samples  math  wait  nsel short  instr')
for r in body:
    print(f"{I(r, 'Warp Stall Sampling (All Samples)'):6d} {I(r, 'stall_math'):5d} {I(r, 'stall_wait'):5d} "
          f"{I(r, 'stall_not_selected'):5d} {I(r, 'stall_short_sb'):5d}  {r[col['Source']].strip()[:80]}")
