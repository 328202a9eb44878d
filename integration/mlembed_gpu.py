"""Reference-side binding: `mlembed._gpu` as a maintainer would add it.

This is the ctypes stub of INTEGRATION.md section 2, kept as a file so the
tests execute it (tests/test_integration.py): it rebinds the reference's
operator boundary -- the numba kernel `mlembed.trainer._train_pass`
(trainer.py:184-207), looked up as a module global by `train_level`
(trainer.py:232) -- to `gb_train_passes` of include/gosh_b200.h.  Host numpy
arrays stay at the API; torch only owns the device memory.

Enable in a process that has `mlembed` importable:

    import mlembed.trainer as t
    from integration import mlembed_gpu as g
    g.enable(t)          # t._train_pass = g._train_pass
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

_LIB = os.environ.get("GB_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
    "paper_2008_12336_b200", "libgosh_b200.so")
_L = C.CDLL(_LIB)
_p, _i64, _u64, _int = C.c_void_p, C.c_int64, C.c_uint64, C.c_int
# int gb_train_passes(V, xadj, adj, sources, n_sources, M, dim, n_neg, seed,
#   rng_stream, pass_begin, n_passes, passes_per_epoch, lr_per_epoch, flags,
#   max_groups, status, stream)                       (include/gosh_b200.h)
_L.gb_train_passes.argtypes = [_i64, _p, _p, _p, _i64, _p, _int, _int, _u64, _u64,
                               _i64, _i64, _i64, _p, C.c_uint, _i64, _p, _p]
_L.gb_train_passes.restype = _int
_L.gb_last_error.restype = C.c_char_p
GB_TRAIN_REUSE, GB_TRAIN_EXACT = 1, 2


def _check(rc):
    if rc:
        raise RuntimeError(_L.gb_last_error().decode())


def _train_pass(xadj, adj, M, lr, n_s, seed, stream, pass_idx, num_workers, reuse):
    """Drop-in for mlembed.trainer._train_pass (trainer.py:184-207): one
    vertex pass over M in place.  num_workers == 1 runs the EXACT kernel
    (bit-equal to the reference's sequential pass); more workers run the
    parallel (Hogwild) kernel, as the reference's prange does."""
    dx = torch.from_numpy(np.ascontiguousarray(xadj, np.int64)).cuda()
    da = torch.from_numpy(np.ascontiguousarray(adj, np.int32)).cuda()
    dM = torch.from_numpy(M).cuda()
    lr_t = torch.tensor([lr], dtype=torch.float32, device="cuda")
    st = torch.tensor([0, 2**63 - 1, 0, 0], dtype=torch.int64, device="cuda")
    flags = (GB_TRAIN_REUSE if reuse else 0) | (GB_TRAIN_EXACT if num_workers == 1 else 0)
    # one pass (pass_idx) of one epoch; lr_per_epoch[pass_idx // ppe] must be
    # lr: passes_per_epoch = pass_idx + 1 maps every pass to entry 0
    _check(_L.gb_train_passes(len(xadj) - 1, dx.data_ptr(), da.data_ptr(), None, 0,
                              dM.data_ptr(), M.shape[1], n_s, seed, stream, pass_idx, 1,
                              pass_idx + 1, lr_t.data_ptr(), flags, 0, st.data_ptr(),
                              torch.cuda.current_stream().cuda_stream))
    M[...] = dM.cpu().numpy()


def enable(trainer_module) -> None:
    """Rebind the reference's kernel name (trainer.py:232 resolves it at
    call time)."""
    trainer_module._train_pass = _train_pass
