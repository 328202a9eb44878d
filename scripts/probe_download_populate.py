"""Download of a large device matrix into a fresh numpy array (measurement
tool): the staged copy as is, and with the destination's pages populated
first by madvise(MADV_POPULATE_WRITE) in parallel slices."""
import ctypes
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2008_12336_b200._staging import copy_device_to_numpy  # noqa: E402

MADV_POPULATE_WRITE = 23
libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]


def populate(a, threads):
    base = a.ctypes.data
    n = a.nbytes
    page = 4096
    start = (base + page - 1) // page * page
    end = (base + n) // page * page
    step = ((end - start) // threads + page - 1) // page * page

    def one(i):
        s = start + i * step
        e = min(end, s + step)
        if e > s:
            r = libc.madvise(s, e - s, MADV_POPULATE_WRITE)
            if r != 0:
                return ctypes.get_errno()
        return 0
    with ThreadPoolExecutor(threads) as ex:
        return list(ex.map(one, range(threads)))


thp = open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()
GB = int(os.environ.get("GB", "31"))
t = torch.empty(GB << 28, dtype=torch.float32, device="cuda")  # GB GiB
t.fill_(1.0)
torch.cuda.synchronize()
for mode in ("plain", "populate8", "populate16", "plain"):
    out = np.empty(t.numel(), dtype=np.float32)
    t0 = time.perf_counter()
    errs = None
    if mode.startswith("populate"):
        errs = populate(out, int(mode[8:]))
    t1 = time.perf_counter()
    copy_device_to_numpy(out, t)
    t2 = time.perf_counter()
    print(json.dumps({"mode": mode, "gib": GB, "thp": thp, "populate_s": t1 - t0,
                      "copy_s": t2 - t1, "total_gbs": out.nbytes / (t2 - t0) / 1e9,
                      "madvise_errno": errs, "ok": bool(out[-1] == 1.0)}), flush=True)
    del out
