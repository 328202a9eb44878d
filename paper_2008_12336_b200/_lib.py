"""ctypes binding of the C ABI in include/gosh_b200.h (libgosh_b200.so).

This is the reference-side binding a maintainer would add: every entry point
takes plain device pointers, sizes and a cudaStream_t.  Device buffers are
torch CUDA tensors (torch is plumbing here: allocation, streams, copies);
the compute is the library's sm_100a kernels.  There is no fallback: a
missing library or a missing GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from .errors import MlembedError

_HERE = os.path.dirname(os.path.abspath(__file__))
# GB_LIB_PATH: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("GB_LIB_PATH") or os.path.join(_HERE, "libgosh_b200.so")

GB_OK = 0
GB_E_INVALID = -1
GB_TRAIN_REUSE = 1
GB_TRAIN_EXACT = 2
GB_TRAIN_FAST_SIGMOID = 4
GB_TRAIN_ATOMIC = 8
GB_CSR_DROP_SELF = 1
GB_CSR_SYMMETRIZE = 2
STATUS_WORDS = 4

_p, _i64, _u64, _int, _dbl, _sz = C.c_void_p, C.c_int64, C.c_uint64, C.c_int, C.c_double, C.c_size_t
_pi64 = C.POINTER(C.c_int64)
_pint = C.POINTER(C.c_int)
_psz = C.POINTER(C.c_size_t)

SIGNATURES = {
    "gb_last_error": (C.c_char_p, []),
    "gb_version": (_int, []),
    "gb_device_info": (_int, [_int, _pint, _pint]),
    "gb_rng_draw_below": (_int, [_u64, _u64, _u64, _u64, _u64, _i64, _i64, _p, _p]),
    "gb_csr_build_workspace": (_int, [_i64, _i64, C.c_uint, _psz]),
    "gb_csr_build": (_int, [_i64, _p, _p, _i64, C.c_uint, _p, _p, _pi64, _p, _sz, _p]),
    "gb_csr_densify_workspace": (_int, [_i64, _psz]),
    "gb_csr_densify": (_int, [_i64, _i64, _p, _p, _p, _p, _p, _p, _pi64, _p, _sz, _p]),
    "gb_rmat_permutation_workspace": (_int, [_int, _psz]),
    "gb_rmat_permutation": (_int, [_int, _u64, _p, _p, _sz, _p]),
    "gb_rmat_edges": (_int, [_int, _i64, _dbl, _dbl, _dbl, _u64, _p, _p, _p, _p]),
    "gb_degree_order_workspace": (_int, [_i64, _psz]),
    "gb_degree_order": (_int, [_i64, _p, _p, _p, _sz, _p]),
    "gb_collapse_workspace": (_int, [_i64, _psz]),
    "gb_collapse": (_int, [_i64, _p, _p, _p, _p, _dbl, _p, _pi64, _pint, _p, _sz, _p]),
    "gb_collapse_cas_workspace": (_int, [_i64, _psz]),
    "gb_collapse_cas": (_int, [_i64, _p, _p, _p, _dbl, _i64, _p, _pi64, _p, _sz, _p]),
    "gb_coarse_csr_workspace": (_int, [_i64, _i64, _i64, _psz]),
    "gb_coarse_csr": (_int, [_i64, _i64, _p, _p, _p, _i64, _p, _p, _pi64, _p, _sz, _p]),
    "gb_expand": (_int, [_p, _i64, _int, _p, _i64, _p, _p]),
    "gb_checksum": (_int, [_p, _i64, _int, _p, _p]),
    "gb_arc_histogram": (_int, [_p, _p, _i64, C.c_uint, _p, _p]),
    "gb_arc_keys_range": (_int, [_p, _p, _i64, C.c_uint, _i64, _i64, _i64, _p, _p, _p]),
    "gb_mapped_histogram": (_int, [_p, _p, _i64, _p, _p, _p]),
    "gb_mapped_keys_range": (_int, [_p, _p, _i64, _p, _i64, _i64, _i64, _p, _p, _p]),
    "gb_mapped_keys_rows": (_int, [_p, _p, _i64, _p, _i64, _i64, _i64, _p, _p, _p, _i64, _i64,
                                   _p]),
    "gb_keys_to_rows_workspace": (_int, [_i64, _i64, _i64, _psz]),
    "gb_keys_to_rows": (_int, [_p, _i64, _i64, _i64, _i64, _p, _p, _pi64, _p, _sz, _p]),
    "gb_rmat_edges_range": (_int, [_int, _i64, _i64, _dbl, _dbl, _dbl, _u64, _p, _p, _p, _p]),
    "gb_csr_validate_workspace": (_int, [_i64, _psz]),
    "gb_csr_validate": (_int, [_i64, _i64, _p, _p, _pint, _p, _sz, _p]),
    "gb_parse_edge_text_workspace": (_int, [_i64, _psz]),
    "gb_parse_edge_text": (_int, [_p, _i64, _p, _p, _pi64, _p, _sz, _p]),
    "gb_unique_ids_workspace": (_int, [_i64, _psz]),
    "gb_unique_ids": (_int, [_p, _i64, _p, _pi64, _int, _p, _sz, _p]),
    "gb_train_passes": (_int, [_i64, _p, _p, _p, _i64, _p, _int, _int, _u64, _u64, _i64, _i64,
                               _i64, _p, C.c_uint, _i64, _p, _p]),
    "gb_train_passes_ppr": (_int, [_i64, _p, _p, _p, _i64, _p, _int, _int, _u64, _u64, _i64,
                                   _i64, _i64, _p, C.c_uint, _i64, _p, _dbl, _p]),
    "gb_active_sources_workspace": (_int, [_i64, _psz]),
    "gb_active_sources": (_int, [_i64, _p, _p, _pi64, _p, _sz, _p]),
    "gb_apply_sample_lists": (_int, [_p, _int, _i64, _p, _int, _p, _p, _dbl, C.c_uint, _i64, _p,
                                     _p]),
    "gb_nonfinite_scan": (_int, [_p, _i64, _i64, _p, _p]),
    "gb_fill_pool_side": (_int, [_p, _p, _i64, _i64, _i64, _i64, _int, _u64, _u64, _p, _p]),
    "gb_train_pool_side": (_int, [_p, _p, _int, _p, _i64, _int, _i64, _i64, _int, _dbl, _u64,
                                  _u64, _p, _p, _i64, _u64, C.c_uint, _i64, _p, _p]),
    "gb_fill_pool_compact": (_int, [_p, _p, _i64, _i64, _i64, _i64, _int, _u64, _u64, _p, _p,
                                    _p, _p]),
    "gb_train_pool_list": (_int, [_p, _p, _int, _p, _p, _p, _i64, _int, _i64, _i64, _int, _dbl,
                                  _u64, _u64, C.c_uint, _i64, _p, _p]),
    "gb_fill_pool_balanced": (_int, [_p, _p, _i64, _i64, _i64, _i64, _i64, _u64, _u64, _p,
                                     _p, _p, _p, _p, _p]),
    "gb_train_pool_balanced": (_int, [_p, _p, _int, _p, _p, _p, _p, _p, _i64, _int, _i64,
                                      _i64, _int, _dbl, _u64, _u64, _p, _i64, _u64, C.c_uint,
                                      _i64, _p, _p]),
    "gb_fill_pool_side_dp": (_int, [_p, _p, _i64, _i64, _i64, _i64, _int, _p, _u64, _p, _p]),
    "gb_train_pool_side_dp": (_int, [_p, _p, _int, _p, _i64, _int, _i64, _i64, _int, _p, _u64,
                                     _p, _p, _i64, _u64, C.c_uint, _i64, _p, _p]),
    "gb_fill_pool_compact_dp": (_int, [_p, _p, _i64, _i64, _i64, _i64, _int, _p, _u64, _p, _p,
                                       _p, _p]),
    "gb_train_pool_list_dp": (_int, [_p, _p, _int, _p, _p, _p, _i64, _int, _i64, _i64, _int, _p,
                                     _u64, C.c_uint, _i64, _p, _p]),
    "gb_fill_pool_balanced_dp": (_int, [_p, _p, _i64, _i64, _i64, _i64, _i64, _p, _u64, _p,
                                        _p, _p, _p, _p, _p]),
    "gb_train_pool_balanced_dp": (_int, [_p, _p, _int, _p, _p, _p, _p, _p, _i64, _int, _i64,
                                         _i64, _int, _p, _u64, _p, _i64, _u64, C.c_uint,
                                         _i64, _p, _p]),
    "gb_host_register": (_int, [_p, _sz]),
    "gb_host_unregister": (_int, [_p]),
    "gb_undirected_pairs_workspace": (_int, [_i64, _psz]),
    "gb_undirected_pairs": (_int, [_p, _p, _i64, _p, _p, _i64, _pi64, _p, _sz, _p]),
    "gb_split_partition_workspace": (_int, [_i64, _i64, _psz]),
    "gb_split_partition": (_int, [_p, _p, _i64, _p, _i64, _i64, _p, _p, _p, _p, _p, _p, _pi64,
                                  _p, _sz, _p]),
    "gb_pairs_member_workspace": (_int, [_i64, _psz]),
    "gb_pairs_member": (_int, [_p, _p, _i64, _p, _p, _i64, _p, _p, _i64, _p, _p, _sz, _p]),
    "gb_hadamard_features": (_int, [_p, _i64, _int, _p, _i64, _p, _p]),
    "gb_logreg_epoch": (_int, [_p, _int, _p, _p, _i64, _int, _dbl, _p, _p, _p]),
    "gb_predict_scores": (_int, [_p, _int, _i64, _p, _dbl, _p, _p]),
    "gb_auc_roc_workspace": (_int, [_i64, _psz]),
    "gb_auc_roc": (_int, [_p, _p, _i64, _p, _p, _sz, _p]),
}

_lib = None


class NativeLibraryError(MlembedError, RuntimeError):
    """The CUDA library is missing or failed."""


def load():
    """Load libgosh_b200.so (no GPU needed to load; every compute call needs one)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (or `make lib`) -- there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def u64(x: int) -> int:
    return int(x) & 0xFFFFFFFFFFFFFFFF


def check(rc: int, what: str) -> None:
    if rc == GB_OK:
        return
    msg = load().gb_last_error().decode(errors="replace")
    if rc == GB_E_INVALID:
        raise ValueError(f"{what}: {msg}")
    raise NativeLibraryError(f"{what} failed ({rc}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise NativeLibraryError("paper_2008_12336_b200 needs a CUDA device (B200); "
                                 "there is no CPU path")
    load()
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "device buffers must be contiguous CUDA tensors"
    return t.data_ptr()


def workspace(query: str, *args) -> tuple[torch.Tensor, int]:
    n = C.c_size_t(0)
    call(query, *args, C.byref(n))
    try:
        ws = torch.empty(max(int(n.value), 1), dtype=torch.uint8, device="cuda")
    except torch.OutOfMemoryError:
        # big-graph workspaces (tens of GiB) can fail on cached-but-fragmented
        # blocks; hand them back to the driver and retry once
        torch.cuda.empty_cache()
        ws = torch.empty(max(int(n.value), 1), dtype=torch.uint8, device="cuda")
    return ws, int(n.value)


def new_status() -> torch.Tensor:
    """[nonfinite flag, first bad epoch, positive updates, reserved]."""
    return torch.tensor([0, 2**63 - 1, 0, 0], dtype=torch.int64, device="cuda")


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
