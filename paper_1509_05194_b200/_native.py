"""ctypes binding of libda_b200.so (the C-ABI declared in include/da_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is visible, every entry point raises RuntimeError.  Status codes follow the
header: < 0 -> ValueError, > 0 -> RuntimeError, message from da_last_error().
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# DA_LIB_PATH: load another in-tree build of the same library (A/B timing runs)
LIB_PATH = os.environ.get("DA_LIB_PATH") or os.path.join(_HERE, "libda_b200.so")

_lock = threading.Lock()
_lib = None

_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_int64

# name -> argtypes (all return int unless noted)
_SIGNATURES = {
    "da_row_sqnorms": [_P, _I, _L, _L, _I, _P, _P],
    "da_assign": [_P, _I, _L, _L, _I, _P, _L, _I, _P, _P, _P, _P, _P, _P, _P],
    "da_group_sums": [_P, _L, _L, _I, _P, _I, _I, _P, _L, _P, _P],
    "da_label_order": [_P, _L, _I, _P, _P, _P],
    "da_gather_rows": [_P, _L, _I, _P, _P, _I, _P, _L, _P],
    "da_heat_up": [_P, _L, _I, _P, _P, _I, _I, _I, _P, _P],
    "da_vec_err": [_P, _I, _L, _L, _I, _P, _I, _L, _P, _I, _I, _P, _P],
    "da_reconstruct": [_P, _I, _L, _L, _P, _I, _I, _I, _P, _P],
    "da_col_mean": [_P, _I, _L, _L, _I, _P, _P],
    "da_pca_cov": [_P, _I, _L, _L, _I, _P, _P, _I, _P],
    "da_col_sums": [_P, _I, _L, _L, _I, _P, _P, _P],
    "da_cov_chains": [_P, _I, _L, _L, _I, _P, _P, _I, _P, _P, _P],
    "da_fold": [_P, _I, _L, _I, _P, _P],
    "da_lloyd_step": [_P, _L, _L, _I, _I, _P, _P, _L, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "da_lloyd_graphs": [_I],
    "da_ctx_create": [_I, _P, _P],
    "da_ctx_stream": [_P, _I, _P],
    "da_nccl_unique_id": [_P],
    "da_ctx_nccl_init": [_P, _I, _I, _P],
    "da_ctx_allreduce_f64": [_P, _P, _L, _P],
    "da_ctx_allgather_i32": [_P, _P, _P, _L, _P],
    "da_ctx_shift_f64": [_P, _P, _P, _L, _P],
    "da_ctx_destroy": [_P],
    "da_lloyd_graph_stats": [_P],
    "da_lloyd_prepare": [_P, _P, _P, _L, _P, _P, _P],
    "da_lloyd_finish": [_I, _P, _P, _I, _I, _P, _L, _P, _P, _P, _P, _P, _L, _L, _P, _P, _P, _P, _P, _P],
    "da_gs_shard_sort": [_P, _L, _L, _I, _P, _I, _P, _P],
    "da_gs_shard_plan": [_P, _L, _L, _I, _I, _P, _I, _I, _L, _P, _P, _P, _I, _P, _P],
    "da_gs_shard_round": [_P, _L, _I, _I, _P, _P, _P, _P],
    "da_gs_shard_fold": [_I, _I, _P, _L, _P, _I, _P, _L, _P],
    "da_rotate": [_P, _I, _L, _L, _I, _P, _P, _P, _I, _P],
    "da_gemm_strided": [_P, _I, _L, _L, _P, _I, _L, _L, _P, _L, _L, _L, _L, _L, _P],
    "da_einsum_sq": [_P, _L, _I, _P, _P],
    "da_cross_products": [_P, _I, _I, _I, _I, _P, _P, _P],
    "da_encode": [_P, _I, _L, _L, _I, _P, _I, _I, _I, _P, _P, _P, _I, _L, _P, _P],
    "da_pair_sums": [_P, _I, _L, _L, _P, _I, _I, _P, _P],
    "da_adc_lut": [_P, _L, _I, _P, _I, _I, _P, _P, _P, _P],
    "da_adc_scan": [_P, _I, _L, _P, _P, _L, _L, _P, _P, _I, _I, _I, _P, _P, _P],
    "da_adc_pack": [_P, _I, _L, _L, _P, _I, _P, _P],
    "da_unpack_vecs": [_P, _L, _I, _I, _P, _L, _P, _P],
    "da_knn": [_P, _I, _L, _L, _I, _P, _P, _L, _P, _I, _P, _P, _P],
    "da_atree_search": [_P, _P, _L, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _L, _L, _L, _L, _P, _I,
                        _P, _P, _P, _P, _P],
    "da_adc_scan_packed": [_P, _P, _L, _L, _P, _P, _I, _I, _I, _P, _P, _P],
    "da_np_sum": [_P, _L, _I, _P, _P],
    "da_select_better": [_L, _I, _P, _P, _P, _P, _P],
    "da_set_column": [_P, _L, _I, _I, _P, _P],
    "da_encode_config": [_I, _P],
    "da_assign_config": [_I, _P],
    "da_assign_bind_image": [_P, _I, _L, _L, _I, _P, _P],
    "da_release_scratch": [],
    "da_prof_enable": [_I],
    "da_prof_collect": [ctypes.c_char_p, _I],
    "da_version": [],
}

EXPORTED = tuple(_SIGNATURES) + ("da_last_error", "da_launch_count", "da_assign_image_bytes")


def launch_count() -> int:
    """Kernels launched by libda_b200 so far in this process."""
    return int(load_library().da_launch_count())


def prof_enable(on: bool) -> None:
    native.da_prof_enable(1 if on else 0)


def prof_collect() -> dict:
    """{kernel name: (launches, total ms)} since the last collect."""
    buf = ctypes.create_string_buffer(1 << 16)
    native.da_prof_collect(buf, len(buf))
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split()
        out[name] = (int(cnt), float(ms))
    return out


def load_library(path: str = LIB_PATH):
    """Load the shared library and declare every export (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"CUDA extension not built: {path} is missing "
                "(run `python -c 'import __graft_entry__ as g; g.build()'` or `make -C "
                "paper_1509_05194_b200/csrc`)"
            )
        lib = ctypes.CDLL(path)
        for name, argtypes in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = ctypes.c_int
        lib.da_launch_count.argtypes = []
        lib.da_launch_count.restype = ctypes.c_longlong
        lib.da_assign_image_bytes.argtypes = [_L, _I]
        lib.da_assign_image_bytes.restype = ctypes.c_int64
        lib.da_last_error.argtypes = []
        lib.da_last_error.restype = ctypes.c_char_p
        _lib = lib
        return lib


def _raise(rc: int, name: str):
    msg = (_lib.da_last_error() or b"").decode(errors="replace")
    if rc < 0:
        raise ValueError(msg or f"{name}: invalid argument")
    raise RuntimeError(f"{name} failed (CUDA status {rc}): {msg}")


class _Caller:
    def __getattr__(self, name):
        lib = load_library()
        fn = getattr(lib, name)

        def call(*args):
            rc = fn(*args)
            if rc != 0:
                _raise(rc, name)
            return rc

        call.__name__ = name
        return call


native = _Caller()
