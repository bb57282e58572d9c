#!/usr/bin/env python3
"""SASS evidence for profiles/: static opcode histograms of the blend kernels (cuobjdump of the
built objects) and, from an `ncu --set full --import-source on` report, the dynamic instruction
mix of each kernel's hottest loop (instructions executed per SASS line).

  python tools/sass_summary.py <report.ncu-rep> <out.json>
"""
import collections
import csv
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OBJS = {"k_blend_fwd": "build/isg/k_blend.o", "k_blend_bwd": "build/isg/k_blend_bwd.o",
        "k_adam_stream": "build/isg/k_adam.o", "k_preprocess": "build/isg/k_preprocess.o"}
CLASSES = {  # opcode -> class
    "FFMA2": "fp32x2", "FMUL2": "fp32x2", "FADD2": "fp32x2", "FFMA": "fp32", "FMUL": "fp32",
    "FADD": "fp32", "MUFU": "mufu", "SHFL": "shuffle", "FSEL": "select", "SEL": "select",
    "LDS": "shared", "STS": "shared", "LDG": "global", "STG": "global", "REDG": "global_red",
    "LDGSTS": "cp.async", "ISETP": "compare", "FSETP": "compare", "VOTE": "vote",
}


def opcode(s):
    t = s.split()
    if not t:
        return None
    op = t[1] if t[0].startswith("@") else t[0]
    return op.split(".")[0]


def static(obj):
    txt = subprocess.run(["cuobjdump", "-sass", str(ROOT / obj)], capture_output=True,
                         text=True).stdout
    out, cur = {}, None
    for line in txt.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            out[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(.*?);", line)
        if cur and m:
            op = opcode(m.group(1))
            if op:
                out[cur][op] += 1
    return out


def dynamic(rep, kernel):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kernel}", "--launch-count", "1"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    if not hdr:
        return None
    body = [r for r in rows[hdr[0] + 1:(hdr[1] if len(hdr) > 1 else None)]
            if len(r) > 6 and r[0].startswith("0x")]
    total = sum(int(r[5]) for r in body)
    counts = collections.Counter(int(r[5]) for r in body)
    # the hottest loop: the execution count carrying the most instructions
    hot_n, hot_k = max(((n, k) for n, k in counts.items()), key=lambda x: x[0] * x[1])
    mix = collections.Counter()
    for r in body:
        if int(r[5]) == hot_n:
            mix[opcode(r[1])] += 1
    cls = collections.Counter()
    for op, c in mix.items():
        cls[CLASSES.get(op, "other")] += c
    return {"warp_instructions_per_launch": total,
            "hot_loop": {"executions": hot_n, "instructions_per_iteration": hot_k,
                         "share_of_launch": hot_n * hot_k / total,
                         "opcodes": dict(mix.most_common()), "classes": dict(cls.most_common())}}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    res = {"source": f"cuobjdump -sass of build/isg/*.o (static) and {rep} source page (dynamic)"}
    for k, obj in OBJS.items():
        st = static(obj)
        res[k] = {"static": {fn: {"instructions": sum(c.values()),
                                  "fp32x2": sum(c[o] for o in ("FFMA2", "FMUL2", "FADD2")),
                                  "mufu": c["MUFU"], "shfl": c["SHFL"],
                                  "redg": c["REDG"], "ldgsts": c["LDGSTS"]}
                             for fn, c in st.items() if k in fn},
                  "dynamic": dynamic(rep, k)}
    json.dump(res, open(out, "w"), indent=1)
    for k in OBJS:
        d = res[k]["dynamic"]
        if d:
            print(k, d["warp_instructions_per_launch"], d["hot_loop"]["instructions_per_iteration"],
                  d["hot_loop"]["classes"])


if __name__ == "__main__":
    main()
