"""Local-memory (LDL/STL) sites of one kernel in a cubin, by innermost
source line (nvdisasm line info): spills and stack arrays on the hot path.

usage: python tools/sass_local.py CUBIN KERNEL_MANGLED_NAME
"""
import collections
import re
import subprocess
import sys

cub, kname = sys.argv[1:3]
out = subprocess.run(["nvdisasm", "-gi", "-c", cub], capture_output=True, text=True).stdout.splitlines()
insec, chain, fresh = False, [], True
cnt = collections.Counter()
src = open("paper_2602_14516_b200/csrc/engine.cuh").read().splitlines()
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
        chain.append((m.group(1).split("/")[-1], int(m.group(2))))
        continue
    if re.match(r"\s*/\*[0-9a-f]{4,}\*/", l):
        fresh = True
        if re.search(r"\b(LDL|STL)\b", l):
            top = chain[0] if chain else ("?", 0)
            cnt[("LDL" if "LDL" in l else "STL", top)] += 1
print("total", sum(cnt.values()))
for (op, (f, ln)), v in cnt.most_common(50):
    t = src[ln - 1].strip()[:70] if f == "engine.cuh" else ""
    print(v, op, f, ln, t)
