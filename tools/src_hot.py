"""Per-source-line totals from an ncu `--page source --csv --print-source cuda,sass` export:
instructions executed and stall samples per CUDA line, hottest first.
  ncu -i rep --page source --csv --kernel-name regex:NAME --print-source cuda,sass > k.csv
  python tools/src_hot.py k.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
files, cur_file, hdr, agg = [], None, None, {}
key = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        key = (cur_file, int(r[0]), r[1].strip()[:70])
        continue
    if key is None or not r[2].startswith("0x"):
        continue
    ie = hdr.get("Instructions Executed")
    ss = hdr.get("Warp Stall Sampling (All Samples)")
    a = agg.setdefault(key, [0, 0])
    a[0] += int(r[ie] or 0)
    a[1] += int(r[ss] or 0)
tot_i = sum(v[0] for v in agg.values())
tot_s = sum(v[1] for v in agg.values())
print(f"total warp instructions {tot_i:,}, stall samples {tot_s:,}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{v[0] / tot_i:6.3f} inst {v[1] / tot_s:6.3f} smp  {k[0]}:{k[1]}  {k[2]}")
