"""Summarise an ncu SASS source page (csv): executed warp-instructions by opcode and the hottest
straight-line blocks (runs of equal execution count).  Usage: sass_hist.py source.csv[.gz] [nblocks]"""
import csv
import gzip
import re
import sys
from collections import Counter

path = sys.argv[1]
f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
rows = list(csv.reader(f))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
ci = hdr.index("Instructions Executed")
si = hdr.index("Source")
wi = hdr.index("Warp Stall Sampling (All Samples)")
ins = []
for r in rows[hdr_i + 1:]:
    if len(r) <= ci or not r[0].startswith("0x"):
        continue
    ins.append((int(r[0], 16), r[si].strip(), int(r[ci] or 0), int(r[wi] or 0)))
base = ins[0][0]
tot = sum(x[2] for x in ins)
samp = sum(x[3] for x in ins)
op = Counter()
for a, s, n, w in ins:
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", s)
    op[m.group(2) if m else s] += n
print(f"total warp instructions {tot:.4e}, stall samples {samp}")
for k, v in op.most_common(25):
    print(f"  {k:12s} {v:.3e} {v / tot:6.1%}")
blocks = []
cur = None
for a, s, n, w in ins:
    if cur and n == cur[2]:
        cur[1] = a
        cur[3] += 1
        cur[4] += w
        cur[5].append(s)
    else:
        cur = [a, a, n, 1, w, [s]]
        blocks.append(cur)
blocks.sort(key=lambda b: -b[2] * b[3])
print("hottest blocks (start offset, n instr, exec count, share of instructions, share of stall samples)")
for b in blocks[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"  0x{b[0] - base:05x} {b[3]:4d} x {b[2]:.3e} = {b[2] * b[3] / tot:6.1%}  stalls {b[4] / max(samp, 1):6.1%}  {b[5][0][:40]} .. {b[5][-1][:40]}")
