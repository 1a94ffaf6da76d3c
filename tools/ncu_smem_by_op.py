"""Shared-memory wavefronts per SASS opcode from an ncu source-page CSV
(--page source --print-source sass): python tools/ncu_smem_by_op.py sass.csv"""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read()
rows = list(csv.reader(io.StringIO(txt[txt.index('"Kernel Name"'):])))
hdr = rows[1]
iA, iE = hdr.index("Source"), hdr.index("Instructions Executed")
iW, iI = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal")
agg = collections.defaultdict(lambda: [0, 0, 0])
for r in rows[2:]:
    try:
        n, w, ideal = int(r[iE]), int(r[iW] or 0), int(r[iI] or 0)
    except (ValueError, IndexError):
        continue
    if not w:
        continue
    op = r[iA].strip().split()
    op = op[1] if op[0].startswith("@") else op[0]
    a = agg[op]
    a[0] += n
    a[1] += w
    a[2] += ideal
tot = sum(a[1] for a in agg.values())
for op, (n, w, ideal) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{op:24s} instr {n:10d}  wavefronts {w:10d} ({100 * w / tot:4.1f}%)  per instr {w / max(n, 1):5.2f}  ideal {ideal / max(n, 1):5.2f}")
