"""Per-source-line instruction counts of one kernel: join an ncu SASS source
page (--page source --csv --print-source sass) with nvdisasm -g line info of
the same cubin.  usage: sass_lines.py ncu_sass.csv cubin kernel_substring"""
import csv, re, subprocess, sys
from collections import Counter, defaultdict

ncu_csv, cubin, ksub = sys.argv[1:4]
rows = list(csv.reader(open(ncu_csv)))
hdr = rows[1]
ei, si = hdr.index("Instructions Executed"), hdr.index("Source")
counts = []
for r in rows[2:]:
    try:
        counts.append((int(r[ei]), r[si].strip()))
    except (ValueError, IndexError):
        pass
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# split functions
funcs = re.split(r"\n\s*\.text\.", dis)
target = [f for f in funcs if f.split(":")[0].find(ksub) >= 0 or ksub in f.split("\n")[0]]
if not target:
    sys.exit("kernel not found")
body = target[0]
line = None
seq = []
for ln in body.split("\n"):
    m = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
    if m:
        line = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        seq.append((line, m.group(2).strip()))
print("ncu instrs", len(counts), "nvdisasm instrs", len(seq), file=sys.stderr)
agg = Counter()
ops = defaultdict(Counter)
for (n, s_ncu), (ln, s_dis) in zip(counts, seq):
    agg[ln] += n
    ops[ln][re.sub(r"^@!?U?P\w+\s+", "", s_dis).split(" ")[0]] += n
tot = sum(agg.values())
for ln, n in agg.most_common(int(sys.argv[4]) if len(sys.argv) > 4 else 40):
    top = ", ".join(f"{k} {v * 100 // max(n, 1)}%" for k, v in ops[ln].most_common(4))
    print(f"{100 * n / tot:5.1f}%  {ln}  [{top}]")
