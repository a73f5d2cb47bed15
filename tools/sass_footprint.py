"""Instruction-footprint view of an ncu SASS source export: per engine
function (innermost inlined frame, via nvdisasm line info), static SASS size,
executed instructions, stall_no_inst samples, and the hot static size (the
instructions executed at least once per 1e-4 of the total).

usage: python tools/sass_footprint.py SASS_CSV CUBIN KERNEL_MANGLED_NAME
"""
import bisect
import collections
import csv
import re
import subprocess
import sys

csv_path, cubin, kname = sys.argv[1:4]
src = open("paper_2602_14516_b200/csrc/engine.cuh").read().splitlines()
starts = []
for i, l in enumerate(src, 1):
    s = l.strip()
    if s.startswith(("return", "if", "for", "while", "//", "}", "else", "case", "const ", "auto ", "#")):
        continue
    m = re.match(r"\s*(?:template<[^>]*>\s*)?(?:PDG_\w+\s+)*(?:static\s+)?(?:__device__\s+)?"
                 r"(?:__forceinline__\s+|__noinline__\s+|inline\s+)?(?:const\s+)?[\w:<>*&]+[\s*&]+(\w+)\([^;]*$", l)
    if m and m.group(1) not in ("if", "for", "while", "switch", "return"):
        starts.append((i, m.group(1)))
idx = [s[0] for s in starts]


def fn(file, line):
    if not file.endswith("engine.cuh"):
        return file.split("/")[-1]
    k = bisect.bisect_right(idx, line) - 1
    return starts[k][1] if k >= 0 else "?"


out = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
insec, chain, fresh, chains = False, [], True, []
for l in out:
    if ".section" in l:
        insec = kname in l and '"ax"' in l
        continue
    if not insec:
        continue
    m = re.match(r'\s*//## File "(.+?)", line (\d+)', l)
    if m:
        if fresh:
            chain, fresh = [], False
        chain.append(fn(m.group(1), int(m.group(2))))
        continue
    if re.match(r"\s*/\*[0-9a-f]{4,}\*/", l):
        fresh = True
        chains.append(list(chain))
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ix["Address"]], 16), int(r[ix["Instructions Executed"]] or 0),
                     int(r[ix["stall_no_inst"]] or 0), int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
    except (ValueError, IndexError, KeyError):
        continue
data.sort()
assert len(data) == len(chains), (len(data), len(chains))
tot = sum(d[1] for d in data)
tni = sum(d[2] for d in data)
tall = sum(d[3] for d in data)
size, ex, ni, hot, samp = (collections.Counter() for _ in range(5))
for (a, n, s, sa), ch in zip(data, chains):
    f = ch[0] if ch else "?"
    size[f] += 1
    ex[f] += n
    ni[f] += s
    samp[f] += sa
    if n * 1e4 >= tot:
        hot[f] += 1
print(f"instructions {len(data)}, hot (>=1e-4 of exec) {sum(hot.values())} = {16 * sum(hot.values()) / 1024:.1f} KB;"
      f" no_inst {100 * tni / max(tall, 1):.1f}% of samples")
print(f"{'function':28s} {'static':>7s} {'hot':>6s} {'exec%':>6s} {'no_inst%':>8s} {'samp%':>6s}")
for f, _ in sorted(hot.items(), key=lambda x: -x[1])[:45]:
    print(f"{f:28s} {size[f]:7d} {hot[f]:6d} {100 * ex[f] / tot:6.2f} {100 * ni[f] / max(tni, 1):8.2f} {100 * samp[f] / max(tall, 1):6.2f}")

if len(sys.argv) > 4:  # hot instructions by inlined call chain (finds duplicated inline copies)
    by = collections.Counter()
    for (a, n, s, sa), ch in zip(data, chains):
        if n * 1e4 >= tot:
            by[" < ".join(ch[: int(sys.argv[4])])] += 1
    for k, v in by.most_common(70):
        print(f"{v:5d} {k}")
