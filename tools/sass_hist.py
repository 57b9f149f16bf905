import csv, sys, re
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ai, si, ei = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
stall = hdr.index("Warp Stall Sampling (All Samples)")
op = Counter(); tot = 0; st = Counter()
seq = []
for r in data:
    try: n = int(r[ei])
    except: continue
    s = r[si].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", s)
    mn = m.group(2) if m else s
    base = mn.split(".")[0]
    op[base] += n; tot += n
    try: st[base] += int(r[stall])
    except: pass
    seq.append((r[ai], s, n))
print("total warp-instr", tot)
for k, v in op.most_common(40): print(f"{k:12s} {v:14d} {100*v/tot:6.2f}%  stall-samples {st[k]}")
