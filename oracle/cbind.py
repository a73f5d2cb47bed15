"""ctypes loader for oracle/build/liboracle.so — the plain-C restatement of the
reference replay (TEST INFRASTRUCTURE ONLY)."""
import ctypes as C
import os

from paper_2602_14516_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")
_lib = None


def available():
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.oracle_run.argtypes = [P(abi.Trace), P(abi.Plan), P(abi.Profile), P(abi.SchedParams), C.c_uint64,
                                 P(abi.RunOutput)]
        L.oracle_last_error.restype = C.c_char_p
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def run(trace, plan, profile, params, seed):
    """Returns a tests.parity.Run-compatible object."""
    from tests.parity import Run, _alloc
    out, dec, ttft, sess = _alloc(trace)
    rc = lib().oracle_run(C.byref(trace), C.byref(plan), C.byref(profile), C.byref(params), seed, C.byref(out))
    if rc:
        raise OracleError(rc, lib().oracle_last_error().decode())
    return Run(out, dec, ttft, sess)
