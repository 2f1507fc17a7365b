"""Summarise an `ncu --page source --print-source sass --csv` dump: per-opcode
instruction share and stall-reason totals (used to write profiles/*.md)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0].startswith("0x")]
I = lambda x: int(x) if x else 0
iS, iI = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot_s = sum(I(r[iS]) for r in data) or 1
tot_i = sum(I(r[iI]) for r in data) or 1
print(f"samples {tot_s} warp-instructions {tot_i}")
st = Counter({c: sum(I(r[h.index(c)]) for r in data) for c in stall_cols})
print("stall reasons:", ", ".join(f"{k[6:]} {100 * v / tot_s:.1f}%" for k, v in st.most_common(8)))
ci, cs = Counter(), Counter()
for r in data:
    t = r[1].split()
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    ci[op] += I(r[iI])
    cs[op] += I(r[iS])
print("top opcodes (inst% / samples%):", ", ".join(f"{op} {100 * ci[op] / tot_i:.1f}/{100 * v / tot_s:.1f}"
                                                  for op, v in cs.most_common(12)))
if len(sys.argv) > 2:
    top = sorted(data, key=lambda r: -I(r[iS]))[: int(sys.argv[2])]
    for r in top:
        reasons = sorted(((I(r[h.index(c)]), c[6:]) for c in stall_cols), reverse=True)[:3]
        print(f"  {r[0][-5:]} {r[1][:50]:50s} {100 * I(r[iS]) / tot_s:5.1f}%  {reasons}")
