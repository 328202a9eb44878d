"""Graph and embedding input/output.

* load_edge_list against the REFERENCE's own results (tests/golden/
  edgelist.npz, make_golden.py make_edgelist): CSR, orig_ids, and for
  malformed texts the exception type, line number and message.  The host
  loop on the CPU; the device parser (gb_parse_edge_text + gb_unique_ids) on
  the GPU, also with chunk boundaries inside the text.
* GSHG / GSHE through pinned staging (load_graph / save_graph /
  load_embedding / save_embedding): byte-identical files, and the device
  validation (gb_csr_validate) raising the reference's messages
  (graph.py:61-77) for each corruption.
"""
from __future__ import annotations

import io

import numpy as np
import pytest

import paper_2008_12336_b200 as gb
from paper_2008_12336_b200 import graph as gmod
from paper_2008_12336_b200.errors import EdgeListParseError


def _texts(g):
    for k in range(int(g["n_text"])):
        yield (bytes(g[f"t{k}_text"]).decode("ascii"), bool(g[f"t{k}_directed"]),
               g[f"t{k}_xadj"], g[f"t{k}_adj"], g[f"t{k}_orig"])


def _errors(g):
    for e in range(int(g["n_err"])):
        yield (bytes(g[f"e{e}_text"]).decode("utf-8"), bytes(g[f"e{e}_kind"]).decode(),
               int(g[f"e{e}_line"]), bytes(g[f"e{e}_msg"]).decode("utf-8"))


def _check_error(text, kind, line, msg):
    if kind == "parse":
        with pytest.raises(EdgeListParseError) as ei:
            gb.load_edge_list(io.StringIO(text))
        assert ei.value.line_number == line and str(ei.value) == msg
    else:
        with pytest.raises(OverflowError) as ei:
            gb.load_edge_list(io.StringIO(text))
        assert str(ei.value) == msg


def test_host_parse_errors_match_reference(golden):
    g = golden("edgelist.npz")
    for text, kind, line, msg in _errors(g):
        if kind == "parse":  # the host loop raises before any CSR is built
            with pytest.raises(EdgeListParseError) as ei:
                gmod._parse_edge_lines_host(io.StringIO(text))
            assert ei.value.line_number == line and str(ei.value) == msg


# -- device -------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [None, 997, 64])
def test_device_edge_list_matches_reference(cuda, golden, monkeypatch, chunk):
    if chunk:
        monkeypatch.setattr(gmod, "EDGE_TEXT_CHUNK", chunk)
    g = golden("edgelist.npz")
    for text, directed, xadj, adj, orig in _texts(g):
        h = gb.load_edge_list(io.StringIO(text), directed=directed)
        assert np.array_equal(h.xadj, xadj) and np.array_equal(h.adj, adj)
        assert np.array_equal(h.orig_ids, orig)


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [None, 500])
def test_device_edge_list_errors_match_reference(cuda, golden, monkeypatch, chunk):
    if chunk:
        monkeypatch.setattr(gmod, "EDGE_TEXT_CHUNK", chunk)
    for args in _errors(golden("edgelist.npz")):
        _check_error(*args)


@pytest.mark.gpu
def test_device_edge_list_error_priority_and_empty(cuda, monkeypatch):
    monkeypatch.setattr(gmod, "EDGE_TEXT_CHUNK", 16)
    # an int64 overflow early and a parse error later: the parse error wins
    text = "1 2\n99999999999999999999 3\n" + "4 5\n" * 10 + "6 7 8\n"
    with pytest.raises(EdgeListParseError) as ei:
        gb.load_edge_list(io.StringIO(text))
    assert ei.value.line_number == 13
    with pytest.raises(gb.EmptyGraphError):
        gb.load_edge_list(io.StringIO("# nothing\n\n   \n"))
    # no trailing newline, CRLF line ends, a non-ASCII comment (host chunk)
    h = gb.load_edge_list(io.StringIO("# café\r\n3 1\r\n1 2"))
    assert np.array_equal(h.orig_ids, [1, 2, 3]) and h.num_edges == 4


@pytest.mark.gpu
def test_gshg_round_trip_through_pinned_staging(cuda, tmp_path):
    g = gb.rmat_graph(14, 1 << 17, 3)
    p1, p2 = str(tmp_path / "dev.gshg"), str(tmp_path / "host.gshg")
    gb.save_graph(g, p1)  # device-resident graph: streamed out
    host = gb.Graph(g.num_vertices, g.num_edges, xadj=g.xadj.copy(), adj=g.adj.copy())
    gb.save_graph(host, p2)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    h = gb.load_graph(p1)
    assert h._xadj is None  # device-backed
    assert np.array_equal(h.xadj, g.xadj) and np.array_equal(h.adj, g.adj)


@pytest.mark.gpu
def test_gshg_device_validation_messages(cuda, tmp_path):
    base = gb.from_edges(np.array([[0, 1], [1, 2], [2, 3], [0, 3]]), num_vertices=5)
    x0, a0 = base.xadj.copy(), base.adj.copy()

    def corrupt(fx=None, fa=None):
        x, a = x0.copy(), a0.copy()
        if fx:
            fx(x)
        if fa:
            fa(a)
        return gb.Graph(5, a.shape[0], xadj=x, adj=a)

    cases = [corrupt(fx=lambda x: x.__setitem__(-1, x[-1] - 1)),
             corrupt(fx=lambda x: x.__setitem__(2, x[3] + 1)),
             corrupt(fa=lambda a: a.__setitem__(0, 7)),
             corrupt(fa=lambda a: a.__setitem__(slice(0, 2), a[0:2][::-1]))]
    for k, bad in enumerate(cases):
        with pytest.raises(ValueError) as want:
            bad.validate()
        p = str(tmp_path / f"bad{k}.gshg")
        gb.save_graph(bad, p)
        with pytest.raises(ValueError) as got:
            gb.load_graph(p)
        assert str(got.value) == str(want.value), k
    # truncated file: the host path's error
    p = str(tmp_path / "ok.gshg")
    gb.save_graph(base, p)
    raw = open(p, "rb").read()
    open(p, "wb").write(raw[:-4])
    with pytest.raises(ValueError):
        gb.load_graph(p)


@pytest.mark.gpu
def test_gshe_round_trip_through_pinned_staging(cuda, tmp_path, monkeypatch):
    import torch
    from paper_2008_12336_b200 import _staging
    monkeypatch.setattr(_staging, "CHUNK", 4096)
    monkeypatch.setattr(_staging, "_pool", [])
    M = torch.randn(1000, 33, device="cuda")
    p1, p2 = str(tmp_path / "d.gshe"), str(tmp_path / "h.gshe")
    gb.save_embedding(M, p1)
    gb.save_embedding(M.cpu().numpy(), p2)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    D = gb.load_embedding(p1, device=True)
    assert D.is_cuda and torch.equal(D, M)
    assert np.array_equal(gb.load_embedding(p1), M.cpu().numpy())


@pytest.mark.gpu
def test_staged_array_transfers_round_trip(cuda, monkeypatch):
    """numpy <-> device through the pinned chunks with threaded host copies
    (Graph uploads/downloads, train_multilevel's result): exact, for sizes
    that are not multiples of the chunk."""
    import torch
    from paper_2008_12336_b200 import _staging
    monkeypatch.setattr(_staging, "CHUNK", 4096)
    monkeypatch.setattr(_staging, "_SMALL", 0)
    monkeypatch.setattr(_staging, "_pool", [])
    rng = np.random.default_rng(2)
    for a in (rng.standard_normal((1000, 33)).astype(np.float32),
              rng.integers(-2**62, 2**62, size=12_345),
              rng.integers(0, 2**31 - 1, size=(7, 999), dtype=np.int32)):
        d = _staging.numpy_to_device(a)
        assert d.is_cuda and d.dtype == torch.from_numpy(a).dtype
        assert np.array_equal(d.cpu().numpy(), a)
        back = _staging.device_to_numpy(d)
        assert back.dtype == a.dtype and np.array_equal(back, a)


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [None, 777])
def test_device_edge_list_from_files(cuda, golden, tmp_path, monkeypatch, chunk):
    """Text files take the byte fast path (read from the file's buffer, no
    decode): the golden texts written with LF and CRLF line ends give the
    reference's graphs and errors; a lone carriage return (a line break under
    universal newlines) or a non-ASCII byte restarts on the text stream."""
    if chunk:
        monkeypatch.setattr(gmod, "EDGE_TEXT_CHUNK", chunk)
    g = golden("edgelist.npz")
    for k, (text, directed, xadj, adj, orig) in enumerate(_texts(g)):
        for nl in ("\n", "\r\n"):
            p = tmp_path / f"t{k}.txt"
            p.write_bytes(text.replace("\n", nl).encode("ascii"))
            with open(p) as f:
                h = gb.load_edge_list(f, directed=directed)
            assert np.array_equal(h.xadj, xadj) and np.array_equal(h.adj, adj), (k, nl)
            assert np.array_equal(h.orig_ids, orig)
    for e, (text, kind, line, msg) in enumerate(_errors(g)):
        p = tmp_path / f"e{e}.txt"
        p.write_bytes(text.encode("utf-8"))
        with open(p, encoding="utf-8") as f:
            if kind == "parse":
                with pytest.raises(EdgeListParseError) as ei:
                    gb.load_edge_list(f)
                assert ei.value.line_number == line and str(ei.value) == msg
            else:
                with pytest.raises(OverflowError):
                    gb.load_edge_list(f)
    # lone CR: Python's text mode splits the line there
    p = tmp_path / "cr.txt"
    p.write_bytes(b"# c\n1 2\r3 4\n5 6\n")
    with open(p) as f:
        h = gb.load_edge_list(f)
    assert np.array_equal(h.orig_ids, [1, 2, 3, 4, 5, 6]) and h.num_edges == 6
