"""ctypes binding of libmpbjac.so (C-ABI declared in include/mpbjac.h).

The product path has no CPU fallback: if the shared library is missing, or
no CUDA device is visible, every compute entry point raises
:class:`BackendUnavailableError` instead of computing something else.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# MPB_LIB: an alternative build of the same library (A/B timing of compile-time
# variants, tools/ab.py); it must still be an in-tree build
LIB_PATH = os.environ.get("MPB_LIB") or os.path.join(_HERE, "libmpbjac.so")

MPB_UNIFORM, MPB_FIXED_LOW, MPB_ADAPTIVE_HL, MPB_ADAPTIVE_LH = 0, 1, 2, 3

SOLVE_OK = 0
SOLVE_BREAKDOWN = 1
SOLVE_INDEF_PRECOND = 2
SOLVE_INDEF_MATRIX = 3
SOLVE_NONFINITE = 4
SOLVE_NARROW_OVERFLOW = 5

#: every symbol include/mpbjac.h declares (checked by the CPU test suite)
EXPORTED = (
    "mpb_version", "mpb_status_string", "mpb_create", "mpb_destroy",
    "mpb_set_stream", "mpb_synchronize", "mpb_launch_count",
    "mpb_plan_tiles_host", "mpb_plan_create", "mpb_plan_destroy",
    "mpb_plan_info", "mpb_csr_matvec_f64", "mpb_csr_matvec_f32",
    "mpb_block_jacobi_sweeps_f64", "mpb_block_jacobi_sweeps_f32",
    "mpb_dot_f64", "mpb_dot_f32", "mpb_norm_sq_f64", "mpb_norm_sq_f32",
    "mpb_narrow_f64_f32", "mpb_widen_f32_f64", "mpb_setup_diag_f64",
    "mpb_setup_diag_f32", "mpb_convert_values_f32", "mpb_bjac_apply_f64",
    "mpb_bjac_apply_f32", "mpb_fmp_apply", "mpb_bjac_inner_apply_f64",
    "mpb_bjac_inner_apply_f32", "mpb_solve_workspace_bytes", "mpb_pcg_solve",
    "mpb_true_relres", "mpb_profile_iteration", "mpb_sell_create",
    "mpb_sell_destroy", "mpb_sell_nnz", "mpb_sell_pack_f64", "mpb_sell_pack_f32",
    "mpb_plan_bind_sell", "mpb_plan_inblock_nnz", "mpb_plan_pack_inblock_f64",
    "mpb_plan_pack_inblock_f32", "mpb_comm_unique_id", "mpb_comm_create",
    "mpb_comm_destroy", "mpb_solve_workspace_bytes_dist", "mpb_pcg_solve_dist",
    "mpb_profile_iteration_dist", "mpb_plan_layout_info", "mpb_plan_offset_slot_info", "mpb_stencil_nnz",
    "mpb_assemble_stencil", "mpb_splitmix64_uniform", "mpb_expand_3t",
    "mpb_row_features", "mpb_tau_histogram", "mpb_vector_stats",
    "mpb_first_violations", "mpb_local_group_create", "mpb_local_group_destroy", "mpb_local_group_stream",
    "mpb_comm_create_local",
)


class BackendUnavailableError(RuntimeError):
    """libmpbjac.so is missing or no CUDA device is usable."""


class MpbCsr(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p),
                ("val64", C.c_void_p), ("val32", C.c_void_p),
                ("sell", C.c_void_p), ("sell_val64", C.c_void_p),
                ("sell_val32", C.c_void_p), ("ib_val64", C.c_void_p),
                ("ib_val32", C.c_void_p), ("op_sell_val64", C.c_void_p),
                ("op_ib_val64", C.c_void_p)]


class MpbHalo(C.Structure):
    _fields_ = [("rank_lo", C.c_int), ("rank_hi", C.c_int),
                ("recv_lo", C.c_int64), ("recv_hi", C.c_int64),
                ("send_lo", C.c_int64), ("send_hi", C.c_int64)]


class MpbSolveOptions(C.Structure):
    _fields_ = [("kind", C.c_int), ("adp_tol", C.c_double), ("k", C.c_int),
                ("t", C.c_int), ("res_tol", C.c_double),
                ("max_iter", C.c_int64), ("true_stride", C.c_int64),
                ("has_x0", C.c_int), ("graph_iters", C.c_int)]


class MpbSolveResult(C.Structure):
    _fields_ = [("converged", C.c_int), ("error", C.c_int),
                ("iterations", C.c_int64), ("err_iteration", C.c_int64),
                ("err_value", C.c_double), ("r0_norm", C.c_double),
                ("final_true_relres", C.c_double),
                ("overflow_count", C.c_int64), ("overflow_index", C.c_int64),
                ("device_seconds", C.c_double),
                ("kernel_launches", C.c_int64)]


_P = C.c_void_p
_I64 = C.c_int64
_I64P = C.POINTER(C.c_int64)
_lib = None
_lock = threading.Lock()


def _declare(L):
    sig = {
        "mpb_version": ([], C.c_int),
        "mpb_status_string": ([C.c_int], C.c_char_p),
        "mpb_create": ([C.c_int, _P, C.POINTER(_P)], C.c_int),
        "mpb_destroy": ([_P], C.c_int),
        "mpb_set_stream": ([_P, _P], C.c_int),
        "mpb_synchronize": ([_P], C.c_int),
        "mpb_launch_count": ([_P], C.c_int64),
        "mpb_plan_tiles_host": ([_I64, _P, _P, _P, C.POINTER(C.c_int)], C.c_int64),
        "mpb_plan_create": ([_P, _I64, _I64, _P, _P, C.POINTER(_P)], C.c_int),
        "mpb_plan_destroy": ([_P], C.c_int),
        "mpb_plan_info": ([_P, _I64P, C.POINTER(C.c_int), _I64P], C.c_int),
        "mpb_plan_layout_info": ([_P, C.POINTER(C.c_int), _I64P], C.c_int),
        "mpb_plan_offset_slot_info": ([_P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
        "mpb_stencil_nnz": ([_I64], C.c_int64),
        "mpb_assemble_stencil": ([_P, _I64, _P, C.c_double, C.c_double, C.c_double, C.c_double, _P, _P, _P],
                                 C.c_int),
        "mpb_splitmix64_uniform": ([_P, C.c_uint64, _I64, C.c_double, C.c_double, _P], C.c_int),
        "mpb_expand_3t": ([_P, _I64, _P, _P, _P, _P, _P, C.c_double, _P, _P, _P], C.c_int),
        "mpb_row_features": ([_P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P], C.c_int),
        "mpb_tau_histogram": ([_P, _I64, _P, C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_int64),
                               C.POINTER(C.c_int64)], C.c_int),
        "mpb_vector_stats": ([_P, _I64, _P, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double),
                              C.POINTER(C.c_double), C.POINTER(C.c_int64)], C.c_int),
        "mpb_first_violations": ([_P, C.c_int, _I64, _P, _P, C.c_double, _P, _I64, _P, _P, _P, C.c_int,
                                  C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
        "mpb_csr_matvec_f64": ([_P, _I64, _P, _P, _P, _P, _P], C.c_int),
        "mpb_csr_matvec_f32": ([_P, _I64, _P, _P, _P, _P, _P], C.c_int),
        "mpb_block_jacobi_sweeps_f64": ([_P, _P, _P, _P, _P, _P, C.c_int, _P, _P, _P, _I64, _I64], C.c_int),
        "mpb_block_jacobi_sweeps_f32": ([_P, _P, _P, _P, _P, _P, C.c_int, _P, _P, _P, _I64, _I64], C.c_int),
        "mpb_dot_f64": ([_P, _P, _I64, _P, _P, C.POINTER(C.c_double)], C.c_int),
        "mpb_dot_f32": ([_P, _P, _I64, _P, _P, C.POINTER(C.c_float)], C.c_int),
        "mpb_norm_sq_f64": ([_P, _P, _I64, _P, C.POINTER(C.c_double)], C.c_int),
        "mpb_norm_sq_f32": ([_P, _P, _I64, _P, C.POINTER(C.c_double)], C.c_int),
        "mpb_narrow_f64_f32": ([_P, _I64, _P, _P, _I64P, _I64P], C.c_int),
        "mpb_widen_f32_f64": ([_P, _I64, _P, _P], C.c_int),
        "mpb_setup_diag_f64": ([_P, _I64, _P, _P, _P, _P, _I64P, _I64P], C.c_int),
        "mpb_setup_diag_f32": ([_P, _I64, _P, _P, _P, _P, _I64P, _I64P], C.c_int),
        "mpb_convert_values_f32": ([_P, _I64, _P, _P, _I64P, _I64P], C.c_int),
        "mpb_bjac_apply_f64": ([_P, _P, C.POINTER(MpbCsr), C.c_int, C.c_int, _P, _P], C.c_int),
        "mpb_bjac_apply_f32": ([_P, _P, C.POINTER(MpbCsr), C.c_int, C.c_int, _P, _P], C.c_int),
        "mpb_fmp_apply": ([_P, _P, C.POINTER(MpbCsr), C.c_int, C.c_int, _P, _P, _I64P, _I64P], C.c_int),
        "mpb_bjac_inner_apply_f64": ([_P, C.POINTER(MpbCsr), _I64, _I64, C.c_int, _P, _P], C.c_int),
        "mpb_bjac_inner_apply_f32": ([_P, C.POINTER(MpbCsr), _I64, _I64, C.c_int, _P, _P], C.c_int),
        "mpb_solve_workspace_bytes": ([_P, _I64], C.c_int64),
        "mpb_pcg_solve": ([_P, _P, C.POINTER(MpbCsr), C.POINTER(MpbSolveOptions), _P, _P, _P, _P, _P, _P,
                           _P, _I64, C.POINTER(MpbSolveResult)], C.c_int),
        "mpb_profile_iteration": ([_P, _P, C.POINTER(MpbCsr), C.POINTER(MpbSolveOptions), _P, _P, _P, _I64,
                                   C.c_int, C.c_int, C.POINTER(C.c_double)], C.c_int),
        "mpb_profile_iteration_dist": ([_P, _P, C.POINTER(MpbCsr), C.POINTER(MpbSolveOptions), _I64, _P, _P,
                                        _P, _I64, C.c_int, C.c_int, C.POINTER(C.c_double)], C.c_int),
        "mpb_sell_create": ([_P, _I64, _P, _P, _P, C.POINTER(_P)], C.c_int),
        "mpb_sell_destroy": ([_P], C.c_int),
        "mpb_plan_bind_sell": ([_P, _P, _P], C.c_int),
        "mpb_plan_inblock_nnz": ([_P], C.c_int64),
        "mpb_plan_pack_inblock_f64": ([_P, _P, _P, _P], C.c_int),
        "mpb_plan_pack_inblock_f32": ([_P, _P, _P, _P], C.c_int),
        "mpb_sell_nnz": ([_P], C.c_int64),
        "mpb_sell_pack_f64": ([_P, _P, _P, _P, _P], C.c_int),
        "mpb_sell_pack_f32": ([_P, _P, _P, _P, _P], C.c_int),
        "mpb_comm_unique_id": ([_P], C.c_int),
        "mpb_comm_create": ([_P, C.c_int, C.c_int, _P, C.POINTER(_P)], C.c_int),
        "mpb_comm_destroy": ([_P], C.c_int),
        "mpb_local_group_create": ([C.c_int, C.c_int, C.POINTER(_P)], C.c_int),
        "mpb_local_group_destroy": ([_P], C.c_int),
        "mpb_local_group_stream": ([_P], _P),
        "mpb_comm_create_local": ([_P, C.c_int, C.POINTER(_P)], C.c_int),
        "mpb_solve_workspace_bytes_dist": ([_P, _I64, _I64], C.c_int64),
        "mpb_pcg_solve_dist": ([_P, _P, C.POINTER(MpbHalo), _P, C.POINTER(MpbCsr), C.POINTER(MpbSolveOptions), _P,
                                _P, _P, _P, _P, _P, _P, _I64, C.POINTER(MpbSolveResult)], C.c_int),
        "mpb_true_relres": ([_P, _P, C.POINTER(MpbCsr), _P, _P, C.c_double, C.POINTER(C.c_double)], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res


def load():
    """The loaded library (no GPU needed just to load it)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise BackendUnavailableError(
                        f"{LIB_PATH} is missing: run __graft_entry__.build() "
                        "(make -C paper_2407_15973_b200/csrc)")
                L = C.CDLL(LIB_PATH)
                _declare(L)
                _lib = L
    return _lib


def check(status: int, what: str = "libmpbjac") -> None:
    if status != 0:
        msg = load().mpb_status_string(int(status)).decode()
        if status < 0:
            raise ValueError(f"{what}: {msg}")
        raise RuntimeError(f"{what}: CUDA error {status}: {msg}")


class Handle:
    """One libmpbjac handle per CUDA device, bound to torch's current stream
    at every call."""

    _per_device: dict = {}

    def __init__(self, device: int, stream=None):
        """stream: a raw cudaStream_t for a private handle (None: torch's
        current stream, the per-device handle of Handle.get)."""
        import torch
        self.device = device
        self.lib = load()
        h = C.c_void_p()
        with torch.cuda.device(device):
            if stream is None:
                stream = torch.cuda.current_stream(device).cuda_stream
            check(self.lib.mpb_create(device, C.c_void_p(stream), C.byref(h)),
                  "mpb_create")
        self.ptr = h

    def __del__(self):
        try:
            if self.ptr and self not in Handle._per_device.values():
                self.lib.mpb_destroy(self.ptr)
                self.ptr = C.c_void_p()
        except Exception:  # interpreter shutdown
            pass

    @classmethod
    def get(cls, device=None) -> "Handle":
        import torch
        if not torch.cuda.is_available():
            raise BackendUnavailableError(
                "no CUDA device visible: the B200 kernels have no CPU fallback")
        if device is None:
            device = torch.cuda.current_device()
        device = int(device)
        h = cls._per_device.get(device)
        if h is None:
            h = cls(device)
            cls._per_device[device] = h
        stream = torch.cuda.current_stream(device).cuda_stream
        check(h.lib.mpb_set_stream(h.ptr, C.c_void_p(stream)), "mpb_set_stream")
        return h

    def launches(self) -> int:
        return int(self.lib.mpb_launch_count(self.ptr))


def ptr(t) -> C.c_void_p:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return C.c_void_p(0)
    return C.c_void_p(t.data_ptr())
