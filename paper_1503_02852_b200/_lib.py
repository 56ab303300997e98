"""ctypes binding of the C ABI (include/rnngraph_b200.h) and the in-tree build.

The shared library is built in-tree (``paper_1503_02852_b200/librnngraph_b200.so``)
by ``build()`` / ``__graft_entry__.build()`` with nvcc for sm_100a.  There is no
fallback: if the library is missing or no sm_100 device is present, engine
calls raise.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "librnngraph_b200.so")
SOURCES = ["csrc/rgb_kernels.cu", "csrc/rgb_tc_gemm.cu", "csrc/rgb_scc.cu", "csrc/rgb_plan.cu", "csrc/rgb_prof.cu",
           "csrc/rgb_comm.cu"]
HEADERS = ["csrc/rgb_types.cuh", "csrc/rgb_kernels.cuh", "csrc/rgb_ew.cuh", "csrc/rgb_prof.cuh", "csrc/rgb_scc.cuh",
           "csrc/rgb_comm.cuh", "../include/rnngraph_b200.h"]
PROF_CATEGORIES = ("ew", "gemm", "gemm_frame", "ew_frame", "dw", "softmax", "inject", "sgd", "transpose", "scc")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]

RGB_OK, RGB_ERR_ENGINE, RGB_ERR_KERNEL, RGB_ERR_CUDA, RGB_ERR_FLOAT = 0, 1, 2, 3, 4

_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_SIGS = {
    "rgb_abi_version": ([], _I),
    "rgb_last_error": ([], ctypes.c_char_p),
    "rgb_plan_create": ([_P, _I64, ctypes.POINTER(_P)], _I),
    "rgb_plan_destroy": ([_P], _I),
    "rgb_plan_workspace_bytes": ([_P, ctypes.POINTER(_I64)], _I),
    "rgb_plan_bind": ([_P, _P], _I),
    "rgb_plan_get_cursor": ([_P, ctypes.POINTER(_I64)], _I),
    "rgb_plan_set_cursor": ([_P, _I64], _I),
    "rgb_forward_chunk": ([_P, _P, _P, _I, _I, _I, _P], _I),
    "rgb_forward_chunk_ids": ([_P, _P, _P, _P, _I, _I, _I, _P], _I),
    "rgb_inject_output_error": ([_P, _P, _I, _I, _I, _I, _P], _I),
    "rgb_read_loss": ([_P, ctypes.POINTER(ctypes.c_double), _P], _I),
    "rgb_check_inputs": ([_P, _P], _I),
    "rgb_read_loss_async": ([_P, _P, _P], _I),
    "rgb_set_injection": ([_P, _P, _I, _P], _I),
    "rgb_get_injection": ([_P, _P, _I, _P], _I),
    "rgb_backward_window": ([_P, _P, _P, _I, _I, _I, _P], _I),
    "rgb_comm_unique_id": ([_P], _I),
    "rgb_comm_init": ([_P, _I, _I, ctypes.POINTER(_P)], _I),
    "rgb_comm_destroy": ([_P], _I),
    "rgb_comm_size": ([_P, ctypes.POINTER(_I), ctypes.POINTER(_I)], _I),
    "rgb_allreduce_grads": ([_P, _P, _I64, _P], _I),
    "rgb_allreduce_f64": ([_P, _P, _I64, _I, _P], _I),
    "rgb_backward_window_allreduce": ([_P, _P, _P, _I, _I, _P, _P], _I),
    "rgb_sgd_update": ([_P, _P, _P, _P, ctypes.c_float, _P], _I),
    "rgb_refresh_transpose": ([_P, _P, _P, _P], _I),
    "rgb_reset_stream": ([_P, _I, _P], _I),
    "rgb_window_view": ([_P, _I, _I64, _I64, ctypes.POINTER(_P), ctypes.POINTER(_I)], _I),
    "rgb_count_nonfinite": ([_P, _I, _I64, _I64, ctypes.POINTER(_I64), _P], _I),
    "rgb_inject_rows": ([_P, _P, _I, _I, _P, _P, _P, _I, _I, _P], _I),
    "rgb_onehot_rows": ([_P, _I, _I, _P, _P], _I),
    "rgb_tape_gather": ([_P, _P, _P, _P, _I, _I, _P], _I),
    "rgb_set_gemm_mode": ([_I], _I),
    "rgb_set_tc_precision": ([_I], _I),
    "rgb_set_scc_mode": ([_I], _I),
    "rgb_set_wavefront": ([_I], _I),
    "rgb_set_frame_loop": ([_I], _I),
    "rgb_gemm_nt": ([_P, _P, _P, _I, _I, _I, _I, _P], _I),
    "rgb_gemm_dw": ([_P, _P, _P, _I, _I, _I, ctypes.c_float, _I, _P], _I),
    "rgb_gemm_nt_tma": ([_P, _P, _P, _P, _I, _I, _I, _P], _I),
    "rgb_set_tc_config": ([_I, _I, _I], _I),
    "rgb_launch_count": ([ctypes.POINTER(_I64)], _I),
    "rgb_profile_enable": ([_I], _I),
    "rgb_profile_collect": ([], _I),
    "rgb_profile_reset": ([], _I),
    "rgb_profile_read": ([_I, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64),
                          ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)], _I),
}
EXPORTS = tuple(_SIGS)


class LibraryMissing(RuntimeError):
    pass


def build(verbose: bool = False, force: bool = False) -> str:
    """nvcc-compile the CUDA sources into the in-tree shared library."""
    srcs = [os.path.join(HERE, s) for s in SOURCES]
    deps = srcs + [os.path.join(HERE, h) for h in HEADERS]
    if not force and os.path.exists(LIB_PATH):
        t = os.path.getmtime(LIB_PATH)
        if all(os.path.getmtime(d) <= t for d in deps):
            return LIB_PATH
    # one nvcc per translation unit in parallel (the tensor-core file alone
    # takes ~2 min), then one link step
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    heads = [os.path.join(HERE, h) for h in HEADERS]
    newest_head = max(os.path.getmtime(h) for h in heads)
    cflags = [f for f in NVCC_FLAGS if f != "-shared"]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), newest_head):
            cmd = ["nvcc", *cflags, "-c", src, "-o", obj + ".tmp"]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True, cwd=HERE)
            os.replace(obj + ".tmp", obj)
        return obj

    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(compile_one, srcs))
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB_PATH + ".tmp", *objs, "-ldl"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=HERE)
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


_lib = None


def lib():
    """The loaded library (raises LibraryMissing when it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(handle, name)
            fn.argtypes = args
            fn.restype = res
        _lib = handle
    return _lib


def check(rc: int, where: str = "") -> None:
    """Map a status code to the reference's exception family."""
    if rc == RGB_OK:
        return
    msg = lib().rgb_last_error().decode(errors="replace")
    if where:
        msg = f"{where}: {msg}"
    if rc == RGB_ERR_ENGINE:
        from .schedule import EngineError
        raise EngineError(msg)
    if rc == RGB_ERR_KERNEL:
        raise KernelError(msg)
    if rc == RGB_ERR_FLOAT:
        raise FloatingPointError(msg)
    raise RuntimeError(msg)


class KernelError(ValueError):
    """Mirror of the reference ``KernelError`` (kernels.py:54-55)."""
