"""The C-ABI library loads, exports every entry point include/pdsim_gpu.h
declares, and its struct layouts match the ctypes mirror (no GPU needed)."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from paper_2602_14516_b200 import abi, native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pdsim_gpu.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^[A-Za-z_][\w\s\*]*?\b(pdsim_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("pdsim_gpu_create", "pdsim_gpu_run", "pdsim_gpu_plan_search", "pdsim_gpu_stage",
                 "pdsim_gpu_search_staged", "pdsim_gen_trace", "pdsim_synth_profile", "pdsim_enumerate_plans"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = native.lib()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.pdsim_abi_version() == native.ABI_VERSION == 3


def test_struct_layouts_match_ctypes():
    probe = ["#include <stdio.h>", "#include <stddef.h>", '#include "pdsim_gpu.h"', "int main(void){"]
    for cname, cls in abi.STRUCTS.items():
        probe.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            probe.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    probe.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "p.c")
        exe = os.path.join(d, "p")
        open(src, "w").write("\n".join(probe))
        subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    got = dict(line.rsplit(" ", 1) for line in out.strip().splitlines())
    for cname, cls in abi.STRUCTS.items():
        assert int(got[cname]) == C.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, (cname, fname)


def test_no_cpu_fallback_without_a_device():
    """Without a B200 the product refuses to run (there is no CPU path)."""
    from tests.conftest import HAS_GPU
    if HAS_GPU:
        pytest.skip("a GPU is present")
    with pytest.raises(native.PdsimError) as e:
        native.Context(0)
    assert e.value.code == abi.ERR_CUDA
