"""A/B kernel timing of several builds of libpdsim_gpu.so on the same box:
alternates runs of a staged search in fresh processes.

usage: python tools/ab.py CONFIG ROUNDS LIB [LIB ...]
LIB_x is a libpdsim_gpu.so, or a directory holding a whole package copy
(paper_2602_14516_b200/ with its .so) when the Python bindings differ too;
LIB@VAR=VALUE[,VAR=VALUE] runs that arm with extra environment variables.
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


def main(libs, rounds=3, cfg="C2", pb="0", pe="-1"):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {spec: [] for spec in libs}
    for _ in range(int(rounds)):
        for spec in libs:
            lib, _, extra = spec.partition("@")
            add = dict(kv.split("=", 1) for kv in extra.split(",") if kv)
            if os.path.isdir(lib):
                env = dict(os.environ, PYTHONPATH=os.path.abspath(lib))
                cwd = os.path.abspath(lib)
            else:
                env = dict(os.environ, PDSIM_LIB=os.path.abspath(lib))
                cwd = root
            env.update(add)
            out = subprocess.run([sys.executable, "-c", CHILD, cfg, pb, pe], cwd=cwd, env=env, capture_output=True,
                                 text=True)
            res[spec].append(float(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else None)
            if out.returncode != 0:
                print(out.stderr[-2000:], file=sys.stderr)
    for lib, v in res.items():
        ok = [x for x in v if x is not None]
        print(cfg, lib, v, "min", min(ok) if ok else None, flush=True)


if __name__ == "__main__":
    # usage: ab.py CONFIG ROUNDS LIB [LIB ...]
    main(sys.argv[3:], rounds=sys.argv[2], cfg=sys.argv[1])
