"""Attributes ncu per-instruction samples/executions (SASS CSV) of the replay
kernel to engine.cuh functions via nvdisasm line info (innermost location,
mapped to the enclosing function by line range)."""
import bisect
import collections
import csv
import re
import subprocess
import sys

csv_path, cubin, kname = sys.argv[1], sys.argv[2], sys.argv[3]
src = open("paper_2602_14516_b200/csrc/engine.cuh").read().splitlines()
starts = []
for i, l in enumerate(src, 1):
    m = re.match(r"\s*(?:PDG_HD|PDG_COLD)\s+(?:static\s+)?[\w:<>*&\s]+?\b(\w+)\(", l)
    if m:
        starts.append((i, m.group(1)))
lines_idx = [s[0] for s in starts]


def func_of(fileline):
    f, n = fileline
    if not f.endswith("engine.cuh"):
        return f.split("/")[-1]
    k = bisect.bisect_right(lines_idx, n) - 1
    return starts[k][1] if k >= 0 else "?"


out = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
ins, loc, insec = [], None, False
for l in out:
    if ".section" in l:
        insec = kname in l and '"ax"' in l
        continue
    if not insec:
        continue
    m = re.match(r'\s*//## File "(.+?)", line (\d+)(.*)', l)
    if m:
        loc = (m.group(1), int(m.group(2)))
        continue
    if re.match(r"\s*/\*[0-9a-f]{4,}\*/", l):
        ins.append(loc)
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    try:
        a = int(r[ix["Address"]], 16)
    except (ValueError, IndexError):
        continue
    data.append((a, int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), int(r[ix["Instructions Executed"]] or 0)))
data.sort()
print(len(ins), len(data))
samp, inst = collections.Counter(), collections.Counter()
for (a, s, n), lc in zip(data, ins):
    f = func_of(lc) if lc else "?"
    samp[f] += s
    inst[f] += n
ts, ti = sum(samp.values()), sum(inst.values())
for f, s in samp.most_common(40):
    print(f"{100 * s / ts:5.1f}% samples {100 * inst[f] / ti:5.1f}% inst  {f}")
