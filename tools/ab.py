"""A/B kernel timing of two builds of libpdsim_gpu.so on the same box:
alternates runs of the staged C2 search in fresh processes.

usage: python tools/ab.py LIB_A LIB_B [rounds] [config] [pair_begin] [pair_end]
LIB_x is a libpdsim_gpu.so, or a directory holding a whole package copy
(paper_2602_14516_b200/ with its .so) when the Python bindings differ too.
"""
import os
import subprocess
import sys

CHILD = r'''
import sys
from paper_2602_14516_b200 import native, workloads
cfg, b, e = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
wl = workloads.CONFIGS[cfg]()
with native.Context(0) as ctx:
    ctx.stage(wl.traces, wl.plans, wl.profile, wl.params)
    ctx.search_staged(wl.seed, b, e)
    ms = [ctx.search_staged(wl.seed, b, e).kernel_ms for _ in range(3)]
print(min(ms))
'''


def main(a, b, rounds=3, cfg="C2", pb="0", pe="-1"):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {a: [], b: []}
    for _ in range(int(rounds)):
        for lib in (a, b):
            if os.path.isdir(lib):
                env = dict(os.environ, PYTHONPATH=os.path.abspath(lib))
                cwd = os.path.abspath(lib)
            else:
                env = dict(os.environ, PDSIM_LIB=os.path.abspath(lib))
                cwd = root
            out = subprocess.run([sys.executable, "-c", CHILD, cfg, pb, pe], cwd=cwd, env=env, capture_output=True,
                                 text=True)
            res[lib].append(float(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else None)
    for lib, v in res.items():
        print(cfg, lib, v, "min", min(x for x in v if x is not None))


if __name__ == "__main__":
    main(*sys.argv[1:])
