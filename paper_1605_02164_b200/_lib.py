"""ctypes loader for libbfvec.so (the C ABI in include/bfvec.h).

Argument marshalling only. There is no CPU fallback: if the in-tree library
is missing, importing the binding raises (build it with
``python paper_1605_02164_b200/build.py``).
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BFVEC_LIB") or os.path.join(_HERE, "libbfvec.so")   # BFVEC_LIB: A/B builds

# names and signatures of every symbol declared in include/bfvec.h
_P, _I, _D, _U64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_uint64
SIGNATURES = {
    "bf_vec_plan": ([_I, _I, _I, _D, _P, _I, _I, _U64, _P], _I),
    "bf_vec_plan_destroy": ([_P], None),
    "bf_vec_sample_freqs": ([_P, _P], _I),
    "bf_vec_get_draws": ([_P, _P, _P, _P, _P], _I),
    "bf_vec_filter": ([_P, _P, _P, _P], _I),
    "bf_vec_filter_host": ([_P, _P, _P, _P], _I),
    "bf_vec_filter_host_async": ([_P, _P, _P, _P], _I),
    "bf_vec_host_sync": ([_P], _I),
    "bf_vec_filter_batch": ([_P, _P, _P, _I, _P], _I),
    "bf_vec_filter_partial": ([_P, _P, _I, _I, _P, _I, _P], _I),
    "bf_vec_normalize": ([_P, _P, _I, _I, _P, _P], _I),
    "bf_vec_filter_rows": ([_P, _P, _I, _I, _I, _I, _P, _P], _I),
    "bf_vec_direct": ([_P, _P, _P, _P], _I),
    "bf_vec_diag": ([_P, _P, _P], _I),
    "bf_vec_mse_sweep": ([_P, _P, _P, _I, _P, _I, _P, _P, _P], _I),
    "bf_vec_srgb_to_lab": ([_P, _P, ctypes.c_longlong, _P], _I),
    "bf_vec_filter_partial_p2p": ([_P, _P, _I, _I, _P, _I, _I, _I, _P], _I),
    "bf_vec_normalize_slots": ([_P, _P, _I, _I, _I, _P, _P], _I),
    "bf_vec_lab_to_srgb": ([_P, _P, ctypes.c_longlong, _P], _I),
    "bf_vec_set_option": ([_P, ctypes.c_char_p, _D], _I),
    "bf_vec_plan_info": ([_P, ctypes.c_char_p, _P], _I),
    "bf_vec_philox4x64_10": ([_P, _P, _P], _I),
    "bf_vec_status_string": ([_I], ctypes.c_char_p),
}

_lib = None


class BfVecError(RuntimeError):
    def __init__(self, status, where=""):
        self.status = status
        super().__init__(f"{where}: {status_string(status)} ({status})")


def load():
    """Load the in-tree libbfvec.so; raise if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libbfvec.so not built ({LIB_PATH}); run "
                              "`python paper_1605_02164_b200/build.py`")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def status_string(status: int) -> str:
    return load().bf_vec_status_string(int(status)).decode()


def check(status: int, where: str) -> int:
    if status < 0:
        raise BfVecError(status, where)
    return status
