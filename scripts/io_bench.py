"""Graph input/output throughput on the GPU box.

GSHG: a friendster-shaped CSR (61.1M vertices, 3.74G arcs, 15.4 GB) written
from HBM (save_graph through pinned chunks) and read back into HBM with the
device validation (load_graph), against the host path the reference uses
(np.fromfile + astype + Graph.validate).  Edge-list text: N_LINES "u v"
lines parsed by gb_parse_edge_text (+ densify + CSR) against the reference's
per-line Python loop (graph.py:143-157) on a 1/20 sample, extrapolated.
Files go to $IO_DIR (default /tmp)."""
import io
import json
import os
import sys
import time

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "backend:cudaMallocAsync")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200 import graph as gmod  # noqa: E402
from paper_2008_12336_b200.graph import array_checksum  # noqa: E402

IO_DIR = os.environ.get("IO_DIR", "/tmp")
SCALE = int(os.environ.get("SCALE", "27"))
SAMPLES = int(os.environ.get("SAMPLES", "1900000000"))
N_LINES = int(os.environ.get("N_LINES", "20000000"))


def main():
    if os.environ.get("SKIP_GSHG"):
        return text_bench()
    g = gb.rmat_graph(SCALE, SAMPLES, 7, densify_ids=True)
    nbytes = 24 + 8 * (g.num_vertices + 1) + 4 * g.num_edges
    path = os.path.join(IO_DIR, "gb_io_bench.gshg")
    x, a = g.device_csr()
    cx, ca = array_checksum(x), array_checksum(a[: g.num_edges])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gb.save_graph(g, path)
    os.sync()
    t_save = time.perf_counter() - t0
    del g, x, a
    torch.cuda.empty_cache()
    os.system(f"sync; echo 3 > /proc/sys/vm/drop_caches 2>/dev/null")
    t0 = time.perf_counter()
    h = gb.load_graph(path)
    torch.cuda.synchronize()
    t_load = time.perf_counter() - t0
    hx, ha = h.device_csr()
    ok = (array_checksum(hx), array_checksum(ha[: h.num_edges])) == (cx, ca)
    del h, hx, ha
    torch.cuda.empty_cache()
    os.system(f"sync; echo 3 > /proc/sys/vm/drop_caches 2>/dev/null")
    # the reference's host path: fromfile + astype + validate (graph.py:203-219)
    import struct
    t0 = time.perf_counter()
    with open(path, "rb") as f:
        f.read(8)
        nv, ne = struct.unpack("<QQ", f.read(16))
        xadj = np.fromfile(f, dtype="<u8", count=nv + 1).astype(np.int64)
        adj = np.fromfile(f, dtype="<u4", count=ne).astype(np.int32)
    t_host_read = time.perf_counter() - t0
    t1 = time.perf_counter()
    gb.Graph(int(nv), int(ne), xadj=xadj, adj=adj).validate()
    t_host_validate = time.perf_counter() - t1
    del xadj, adj
    os.remove(path)
    print(json.dumps({"what": "GSHG", "bytes": nbytes, "vertices": int(nv), "arcs": int(ne),
                      "device_save_s": t_save, "device_save_gbs": nbytes / t_save / 1e9,
                      "device_load_validate_s": t_load,
                      "device_load_gbs": nbytes / t_load / 1e9, "round_trip_equal": ok,
                      "host_read_astype_s": t_host_read, "host_validate_s": t_host_validate,
                      "note": "page cache dropped before each read when permitted"}),
          flush=True)
    text_bench()


def text_bench():
    # edge-list text
    rng = np.random.default_rng(3)
    u = rng.integers(0, 1 << 26, size=N_LINES)
    v = rng.integers(0, 1 << 26, size=N_LINES)
    text = "\n".join(f"{p} {q}" for p, q in zip(u.tolist(), v.tolist())) + "\n"
    t0 = time.perf_counter()
    gd = gb.load_edge_list(io.StringIO(text))
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0
    tpath = os.path.join(IO_DIR, "gb_io_bench.txt")
    with open(tpath, "w") as f:
        f.write(text)
    os.system("sync; echo 3 > /proc/sys/vm/drop_caches 2>/dev/null")
    t0 = time.perf_counter()
    with open(tpath) as f:
        gf = gb.load_edge_list(f)
    torch.cuda.synchronize()
    t_file = time.perf_counter() - t0
    same = bool(np.array_equal(gf.orig_ids, gd.orig_ids)) and gf.num_edges == gd.num_edges
    os.remove(tpath)
    sample = "\n".join(text.split("\n", N_LINES // 20)[: N_LINES // 20]) + "\n"
    t0 = time.perf_counter()
    gmod._parse_edge_lines_host(io.StringIO(sample))
    t_host = (time.perf_counter() - t0) * 20
    print(json.dumps({"what": "edge-list text", "lines": N_LINES, "chars": len(text),
                      "vertices": gd.num_vertices, "arcs": gd.num_edges,
                      "device_parse_densify_csr_s": t_dev,
                      "device_lines_per_s": N_LINES / t_dev,
                      "file_byte_path_s": t_file, "file_lines_per_s": N_LINES / t_file,
                      "file_equals_stringio": same,
                      "host_loop_s_extrapolated": t_host,
                      "host_loop_sample_lines": N_LINES // 20}), flush=True)


if __name__ == "__main__":
    main()
