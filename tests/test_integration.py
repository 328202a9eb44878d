"""INTEGRATION.md section 2 executed: the reference-side ctypes stub
(integration/mlembed_gpu.py) that rebinds mlembed.trainer._train_pass
(trainer.py:184-207) to gb_train_passes.

CPU: the stub loads the library, its argtypes match the header's
declaration, and (where the reference is importable, i.e. the build
container) its signature is the numba kernel's.  GPU: the stub, called the
way train_level calls _train_pass (one call per pass, num_workers=1),
reproduces the reference's own train_pass.npz fixtures bit for bit.
"""
from __future__ import annotations

import inspect
import os
import re
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/pkg/src"


def _header_params(name):
    with open(os.path.join(ROOT, "include", "gosh_b200.h")) as f:
        text = f.read()
    m = re.search(r"int\s+" + name + r"\s*\(([^;]*)\);", text)
    assert m, name
    return [p.strip() for p in m.group(1).split(",")]


def test_stub_loads_and_matches_header():
    from integration import mlembed_gpu as stub
    assert hasattr(stub._L, "gb_train_passes")
    assert len(stub._L.gb_train_passes.argtypes) == len(_header_params("gb_train_passes"))


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present")
def test_stub_signature_is_the_reference_kernel():
    sys.path.insert(0, REF_SRC)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    try:
        import mlembed.trainer as t
    except Exception as e:  # numba missing etc.
        pytest.skip(f"mlembed not importable: {e}")
    finally:
        sys.path.remove(REF_SRC)
    from integration import mlembed_gpu as stub
    ref = inspect.signature(getattr(t._train_pass, "py_func", t._train_pass))
    assert list(ref.parameters) == list(inspect.signature(stub._train_pass).parameters)
    assert "_train_pass" in vars(t)  # the name train_level resolves at call time


@pytest.mark.gpu
def test_stub_reproduces_reference_train_passes(cuda, golden):
    from integration import mlembed_gpu as stub
    g = golden("train_pass.npz")
    names = sorted({k.split("_")[0] for k in g if k.startswith("g") and k.endswith("_xadj")})
    graphs = {int(n[1:]): (g[f"{n}_xadj"], g[f"{n}_adj"]) for n in names}
    for k, (gi, d, n_neg, reuse, seed, stream, lr) in enumerate(g["cases"].tolist()):
        xadj, adj = graphs[int(gi)]
        M = g[f"c{k}_M0"].copy()
        for p in range(3):
            stub._train_pass(xadj, adj, M, np.float32(lr), int(n_neg), int(seed), int(stream),
                             p, 1, bool(reuse))
        assert np.array_equal(M, g[f"c{k}_M3"]), k
