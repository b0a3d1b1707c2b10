"""ctypes binding of the C-ABI in ``include/armt_b200.h``.

This is the Python side of the drop-in boundary: plain pointers, sizes and a
``cudaStream_t``. Nonzero status codes become the reference's exception
types. There is deliberately no fallback: if ``libarmt_b200.so`` is missing
or a launch fails, the call raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import DeviceError, DimensionError, InputError

HERE = os.path.dirname(os.path.abspath(__file__))
# ARMT_LIB_PATH: load an experimental build of the same C-ABI (A/B runs)
LIB_PATH = os.environ.get("ARMT_LIB_PATH") or os.path.join(HERE, "libarmt_b200.so")

MAX_MEMBERS = 128
F32, BF16 = 0, 1
EPI_STORE, EPI_RESIDUAL, EPI_RETRIEVE, EPI_SWIGLU, EPI_ROPE, EPI_LSE, EPI_DPFP = 0, 1, 2, 3, 4, 5, 6

# Every symbol the header declares (checked by tests/test_boundary.py).
EXPORTS = ("armt_gemm", "armt_embed", "armt_rmsnorm", "armt_dpfp_den", "armt_attention",
           "armt_rope", "armt_swiglu", "armt_mem_fold", "armt_fold_workspace_bytes", "armt_cast",
           "armt_logits_nll", "armt_last_error", "armt_version", "armt_num_sms",
           "armt_kernel_count", "armt_abi_sizeof", "armt_mem_fold_tc", "armt_fold_tc_workspace_bytes",
           "armt_memop_rows", "armt_lse_finalize", "armt_lse_reduce", "armt_gemm_prof", "armt_embed_bad_ids")

_I = ctypes.c_int
_LL = ctypes.c_longlong
_P = ctypes.c_void_p
_F = ctypes.c_float


class ArmtMembers(ctypes.Structure):
    _fields_ = [("G", _I), ("slot", _I * MAX_MEMBERS), ("layer", _I * MAX_MEMBERS)]


class ArmtGemmArgs(ctypes.Structure):
    _fields_ = [
        ("G", _I), ("M", _I), ("N", _I), ("K", _I),
        ("ab_dtype", _I),
        ("A", _P), ("lda", _LL), ("a_stride", _LL),
        ("B", _P), ("ldb", _LL), ("b_stride", _LL),
        ("C", _P), ("ldc", _LL), ("c_stride", _LL), ("c_dtype", _I),
        ("epilogue", _I),
        ("R", _P), ("ldr", _LL), ("r_stride", _LL),
        ("C2", _P), ("ldc2", _LL), ("c2_stride", _LL),
        ("c2_split", _I),
        ("ssq_out", _P), ("ssq_in", _P), ("ssq_stride", _LL), ("ssq_np", _I),
        ("norm_d", _I), ("norm_eps", _F),
        ("lse_part", _P), ("lse_ld", _LL), ("targets", _P), ("lse_tgt", _P), ("lse_rows", _I),
        ("den", _P), ("den_stride", _LL),
        ("eps", _F),
        ("rope_cos", _P), ("rope_sin", _P),
        ("head_dim", _I), ("rope_cols", _I),
        ("swiglu_block", _I),
        ("max_ctas", _I),
        ("z", _P), ("nu", _I),
        ("a_kwrap", _I), ("b_kwrap", _I),
        ("a_slot", _I * MAX_MEMBERS),
        ("b_index", _I * MAX_MEMBERS),
        ("c_slot", _I * MAX_MEMBERS),
        ("e_index", _I * MAX_MEMBERS),
    ]


_lib = None


def load(path: str = LIB_PATH):
    """Load the library (raises DeviceError if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise DeviceError(f"CUDA extension not built: {path} missing "
                          "(run `python -m paper_2506_05229_b200._build`)")
    lib = ctypes.CDLL(path)
    sig = {
        "armt_gemm": (_I, [ctypes.POINTER(ArmtGemmArgs), _P]),
        "armt_embed": (_I, [_P, _P, _P, _I, _P, _P, _I, _I, _I, _I, _P]),
        "armt_embed_bad_ids": (_LL, [_I]),
        "armt_rmsnorm": (_I, [ctypes.POINTER(ArmtMembers), _P, _LL, _P, _P, _I, _LL, _I, _I, _F, _P]),
        "armt_dpfp_den": (_I, [ctypes.POINTER(ArmtMembers), _P, _LL, _P, _P, _I, _LL, _LL, _P, _LL,
                               _I, _I, _I, _P]),
        "armt_attention": (_I, [_I, _P, _LL, _LL, _P, _LL, _LL, _I, _I, _I, _I, _F, _P]),
        "armt_rope": (_I, [_I, _P, _LL, _LL, _I, _I, _I, _I, _P, _P, _P]),
        "armt_swiglu": (_I, [_I, _P, _LL, _LL, _P, _LL, _LL, _I, _I, _I, _I, _P]),
        "armt_mem_fold": (_I, [ctypes.POINTER(ArmtMembers), _P, _LL, _LL, _I, _I, _I, _P, _P, _P, _LL,
                               _I, _I, _I, _I, _F, _P, _P]),
        "armt_fold_workspace_bytes": (_LL, [_I, _I, _I]),
        "armt_mem_fold_tc": (_I, [ctypes.POINTER(ArmtMembers), _P, _LL, _LL, _I, _I, _I, _P, _P, _P,
                                  _I, _I, _I, _I, _F, _P, _P]),
        "armt_fold_tc_workspace_bytes": (_LL, [_I, _I, _I, _I]),
        "armt_memop_rows": (_LL, [_I, _I]),
        "armt_lse_finalize": (_I, [_P, _LL, _I, _P, _P, _P, _LL, _P]),
        "armt_lse_reduce": (_I, [_P, _LL, _I, _P, _LL, _P]),
        "armt_gemm_prof": (_I, [_P, _I]),
        "armt_cast": (_I, [_P, _I, _P, _I, _LL, _P]),
        "armt_logits_nll": (_I, [_P, _I, _LL, _P, _P, _LL, _I, _P]),
        "armt_last_error": (ctypes.c_char_p, []),
        "armt_version": (ctypes.c_char_p, []),
        "armt_num_sms": (_I, []),
        "armt_kernel_count": (_I, []),
        "armt_abi_sizeof": (_LL, [_I]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if (lib.armt_abi_sizeof(0) != ctypes.sizeof(ArmtGemmArgs)
            or lib.armt_abi_sizeof(1) != ctypes.sizeof(ArmtMembers)
            or lib.armt_abi_sizeof(2) != ArmtGemmArgs.a_slot.offset):
        raise DeviceError("libarmt_b200.so ABI does not match the ctypes binding; rebuild")
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = f"{what}: {load().armt_last_error().decode(errors='replace')}"
    if rc == 1:
        raise DimensionError(msg)
    if rc == 2:
        raise InputError(msg)
    raise DeviceError(msg)


def members(slots, layers) -> ArmtMembers:
    m = ArmtMembers()
    m.G = len(layers)
    if not 1 <= m.G <= MAX_MEMBERS:
        raise DimensionError(f"group of {m.G} members outside 1..{MAX_MEMBERS}")
    for g, (s, l) in enumerate(zip(slots, layers)):
        m.slot[g] = int(s)
        m.layer[g] = int(l)
    return m


def kernel_count() -> int:
    return load().armt_kernel_count()
