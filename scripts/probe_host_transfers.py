"""Host<->device transfer strategies for a 1.34 GB float32 matrix (C3's
finest level): torch .cpu() (pageable, fresh pages), pinned staging chunks
into np.empty, the same into a hugepage-advised mmap, and cudaHostRegister of
the destination; H2D: torch .cuda() from pageable vs staged chunks."""
import json
import mmap
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

N = 2616991 * 128
M = torch.randn(N, device="cuda")
torch.cuda.synchronize()
CH = 64 << 20
pins = [torch.empty(CH, dtype=torch.uint8).pin_memory() for _ in range(2)]


def staged_d2h(dst_u8, src_u8):
    n = src_u8.numel()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    evs = [None, None]
    k = 0
    off = 0
    pend = []
    while off < n:
        m = min(CH, n - off)
        b = pins[k % 2]
        with torch.cuda.stream(side):
            b[:m].copy_(src_u8[off:off + m], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        pend.append((ev, b, off, m))
        if len(pend) == 2:
            e, bb, o, mm = pend.pop(0)
            e.synchronize()
            dst_u8[o:o + mm] = bb.numpy()[:mm]
        off += m
        k += 1
    for e, bb, o, mm in pend:
        e.synchronize()
        dst_u8[o:o + mm] = bb.numpy()[:mm]


def hugepage_array(nbytes):
    mm = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    if hasattr(mmap, "MADV_HUGEPAGE"):
        mm.madvise(mmap.MADV_HUGEPAGE)
    return np.frombuffer(mm, dtype=np.uint8)


res = {}
for rep in range(3):
    t = time.perf_counter()
    a = M.cpu().numpy()
    res.setdefault("torch_cpu", []).append(time.perf_counter() - t)
    del a
    t = time.perf_counter()
    d = np.empty(N * 4, dtype=np.uint8)
    staged_d2h(d, M.view(torch.uint8))
    res.setdefault("staged_np_empty", []).append(time.perf_counter() - t)
    del d
    t = time.perf_counter()
    d = hugepage_array(N * 4)
    staged_d2h(d, M.view(torch.uint8))
    res.setdefault("staged_hugepage", []).append(time.perf_counter() - t)
    del d
    t = time.perf_counter()
    d = np.empty(N * 4, dtype=np.uint8)
    d[::4096] = 0  # fault the pages in
    cudart = torch.cuda.cudart()
    r = cudart.cudaHostRegister(d.ctypes.data, d.nbytes, 0)
    torch.from_numpy(d).copy_(M.view(torch.uint8))
    torch.cuda.synchronize()
    cudart.cudaHostUnregister(d.ctypes.data)
    res.setdefault("register_dst", []).append(time.perf_counter() - t)
    del d
    host = np.random.rand(N).astype(np.float32)
    t = time.perf_counter()
    x = torch.from_numpy(host).cuda()
    torch.cuda.synchronize()
    res.setdefault("h2d_torch_cuda", []).append(time.perf_counter() - t)
    del x
print(json.dumps({"bytes": N * 4, "seconds": res,
                  "thp": open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()}))
