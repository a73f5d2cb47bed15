"""Maps ncu per-instruction stall samples (--page source --print-source sass
CSV) to source lines using nvdisasm line info of the same cubin.

usage: python tools/sass_hotspots.py <sass.csv> <cubin> [top]
"""
import collections
import csv
import re
import subprocess
import sys


def parse_nvdisasm(cubin):
    out = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    loc = None
    for line in out.splitlines():
        m = re.match(r"\s*\.section\s+\.text\.(\S+?),", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            loc = None
            continue
        m = re.match(r"\s*//## File \"(.+?)\", line (\d+)(.*)", line)
        if m:
            f = m.group(1).split("/")[-1]
            inl = ""
            mi = re.search(r"inlined at \"(.+?)\", line (\d+)", m.group(3))
            loc = f"{f}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", line)
        if m and cur:
            funcs[cur].append((int(m.group(1), 16), m.group(2).strip(), loc))
    return funcs


def norm(s):
    return re.sub(r"\s+", " ", s.strip().rstrip(";")).replace("`", "")


def main(csv_path, cubin, top=60):
    rows = list(csv.reader(open(csv_path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        try:
            a = int(r[ix["Address"]], 16)
        except ValueError:
            continue
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        n = int(r[ix["Instructions Executed"]] or 0)
        data.append((a, norm(r[ix["Source"]]), s, n, r))
    data.sort()
    funcs = parse_nvdisasm(cubin)
    # contiguous runs in the CSV -> functions by instruction-text match
    runs = []
    start = 0
    for k in range(1, len(data) + 1):
        if k == len(data) or data[k][0] - data[k - 1][0] > 0x10:
            runs.append(data[start:k])
            start = k
    keyed = {}
    for name, ins in funcs.items():
        keyed[name] = [norm(t) for _, t, _ in ins]
    by_line = collections.Counter()
    by_line_n = collections.Counter()
    by_func = collections.Counter()
    stalls = collections.defaultdict(collections.Counter)
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    unmatched = 0
    for run in runs:
        # find the function whose instruction list matches this run best
        text = [t for _, t, _, _, _ in run]
        best, score = None, -1
        for name, ks in keyed.items():
            if len(ks) != len(text):
                continue
            sc = sum(1 for x, y in zip(ks[:64], text[:64]) if x.split(" ")[0] == y.split(" ")[0])
            if sc > score:
                best, score = name, sc
        if best is None:
            unmatched += sum(x[2] for x in run)
            continue
        ins = funcs[best]
        for (a, t, s, n, r), (off, _, loc) in zip(run, ins):
            by_line[loc] += s
            by_line_n[loc] += n
            by_func[best] += s
            for c in cols:
                v = r[ix[c]]
                if v:
                    stalls[loc][c[6:]] += int(v)
    total = sum(by_line.values()) + unmatched
    print(f"total samples {total} (unmatched {unmatched})")
    for f, s in by_func.most_common(20):
        print(f"{s:8d} {100*s/total:5.1f}%  {f[:120]}")
    print()
    for loc, s in by_line.most_common(int(top)):
        st = ", ".join(f"{k}={v}" for k, v in stalls[loc].most_common(3))
        print(f"{s:8d} {100*s/total:5.1f}%  inst={by_line_n[loc]:9d}  {loc}  [{st}]")


if __name__ == "__main__":
    main(*sys.argv[1:])
