"""Generate golden vectors from the REFERENCE implementation (mlembed).

Run in the build container, where the read-only reference is importable:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports /root/reference/pkg/src/mlembed (and the reference's own test
graph generators, /root/reference/pkg/tests/synth.py) and writes small .npz
fixtures next to this script.  The fixtures travel with the repo; nothing on
the GPU box reads /root/reference.  Every deterministic hot-path result is
captured with num_workers=1 (the reference's only deterministic mode).
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import mlembed as ml  # noqa: E402
from mlembed import _rng  # noqa: E402
from mlembed import bigtrain, coarsen, trainer  # noqa: E402
import synth  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle  # noqa: E402  (only for the R-MAT input, which the reference lacks)


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def pack_graphs(prefix, graphs, out):
    for i, g in enumerate(graphs):
        out[f"{prefix}{i}_xadj"] = np.asarray(g.xadj, dtype=np.int64)
        out[f"{prefix}{i}_adj"] = np.asarray(g.adj, dtype=np.int32)


def rmat_ref_graph(scale, samples, seed, dens):
    x, a = oracle.rmat_graph(scale, samples, seed, densify_ids=dens)
    return ml.Graph(num_vertices=len(x) - 1, num_edges=int(x[-1]), xadj=x, adj=a)


def graphs_for_training():
    return {
        "tiny8": synth.gnp_graph(8, 0.5, seed=2),       # frequent self/duplicate samples
        "gnp60": synth.gnp_graph(60, 0.1, seed=3),
        "path12": synth.path_graph(12),
        "cl300": synth.chung_lu_graph(300, 900, 2.5, seed=5),
        "iso": ml.from_edges([(0, 1), (1, 2), (4, 5)], num_vertices=8),  # isolated 3,6,7
    }


def make_rng():
    rows = []
    for seed in (0, 1, 7, 2**63 + 5, 123456789012345):
        for stream in (0, 1, 3, 2**40):
            for step in (0, 1, 17, 2**33):
                for v in (0, 1, 999, 2**31 - 1):
                    key = int(_rng.stream_key(np.uint64(seed), np.uint64(stream),
                                              np.uint64(step), np.uint64(v)))
                    for ctr in (0, 1, 5):
                        for n in (1, 2, 7, 1000, 2**31 - 1, 2**40 + 3):
                            d = int(_rng.draw_below(np.uint64(key), np.uint64(ctr), np.int64(n)))
                            rows.append((seed, stream, step, v, ctr, n, key, d))
    arr = np.asarray(rows, dtype=np.uint64)
    mix_in = np.asarray([0, 1, 2**64 - 1, 0x9E3779B97F4A7C15, 12345], dtype=np.uint64)
    mix_out = np.asarray([int(_rng.mix64(np.uint64(z))) for z in mix_in], dtype=np.uint64)
    save("rng.npz", table=arr, mix_in=mix_in, mix_out=mix_out)


def make_update():
    rng = np.random.default_rng(11)
    out = {}
    cases = []
    k = 0
    for d in (1, 2, 5, 8, 16, 33, 128):
        for b in (0, 1):
            for reuse in (False, True):
                for self_ in (False, True):
                    M = (rng.random((3, d)) - 0.5).astype(np.float32)
                    if k % 3 == 0:
                        M *= 8.0  # reach the sigmoid clamp
                    v, s = (1, 1) if self_ else (0, 2)
                    lr = float(rng.choice([0.025, 0.25, 0.5]))
                    before = M.copy()
                    trainer.update_embedding(M, v, s, b, lr, reuse_updated_source=reuse)
                    out[f"c{k}_before"] = before
                    out[f"c{k}_after"] = M
                    cases.append((d, b, int(reuse), v, s, lr))
                    k += 1
    out["cases"] = np.asarray(cases, dtype=np.float64)
    save("update.npz", **out)


def make_train_pass():
    out = {}
    cases = []
    k = 0
    for gname, g in graphs_for_training().items():
        for d in (8, 16, 32, 33, 128):
            for n_neg, reuse in ((3, False), (0, False), (5, True)):
                if gname in ("path12", "iso") and d not in (8, 33):
                    continue
                seed, stream = 3 + k, k % 4
                M = trainer.init_embedding(g.num_vertices, d, seed=seed)
                out[f"c{k}_M0"] = M.copy()
                lr = np.float32(0.035)
                for p in range(3):
                    trainer._train_pass(g.xadj, g.adj, M, lr, n_neg, seed, stream, p, 1, reuse)
                out[f"c{k}_M3"] = M.copy()
                cases.append((list(graphs_for_training()).index(gname), d, n_neg, int(reuse),
                              seed, stream, float(lr)))
                k += 1
    pack_graphs("g", list(graphs_for_training().values()), out)
    out["cases"] = np.asarray(cases, dtype=np.float64)
    # train_level: lr decay, edge-scaled passes, counts
    lvl = []
    for j, (gname, unit, e_i, d) in enumerate((("gnp60", "edge-scaled", 3, 16),
                                               ("cl300", "vertex-pass", 4, 32),
                                               ("tiny8", "edge-scaled", 5, 8))):
        g = graphs_for_training()[gname]
        cfg = ml.TrainConfig(dim=d, total_epochs=e_i, seed=9 + j, epoch_unit=unit,
                             negative_samples=3, learning_rate=0.05)
        M = trainer.init_embedding(g.num_vertices, d, seed=9 + j)
        out[f"L{j}_M0"] = M.copy()
        st = trainer.train_level(g, M, cfg, e_i, rng_stream=j + 1)
        out[f"L{j}_M"] = M.copy()
        lvl.append((list(graphs_for_training()).index(gname), d, e_i, 9 + j, j + 1,
                    1 if unit == "edge-scaled" else 0, st.passes, st.updates))
    out["levels"] = np.asarray(lvl, dtype=np.int64)
    save("train_pass.npz", **out)


def coarsen_graphs():
    gs = {
        "gnp70": synth.gnp_graph(70, 0.1, seed=100),
        "gnp300": synth.gnp_graph(300, 0.03, seed=11),
        "star5": synth.star_graph(5),
        "path4": synth.path_graph(4),
        "path50": synth.path_graph(50),
        "twohubs": ml.from_edges([(0, 1), (0, 2), (0, 3), (1, 4), (1, 5)], num_vertices=6),
        "k60": synth.complete_graph(60),
        "match256": synth.matching_graph(256),
        "edgeless50": synth.edgeless_graph(50),
        "cl4000": synth.chung_lu_graph(4000, 12000, 2.5, seed=41),
        "planted": synth.planted_graph(4, 30, 0.3, 0.2, seed=6),
        "small": ml.from_edges(np.asarray([(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5),
                                           (2, 3)]), num_vertices=6),
        "rmat12d": rmat_ref_graph(12, 1 << 15, 7, True),
        "rmat12raw": rmat_ref_graph(12, 1 << 15, 7, False),
    }
    return gs


def make_coarsen():
    out = {}
    names = []
    for i, (name, g) in enumerate(coarsen_graphs().items()):
        names.append(name)
        out[f"g{i}_xadj"] = g.xadj
        out[f"g{i}_adj"] = g.adj
        order = coarsen.degree_order(g)
        out[f"g{i}_order"] = order
        m = coarsen.collapse_map(g, order)
        out[f"g{i}_map"] = m.map
        out[f"g{i}_nc"] = np.int64(m.num_clusters)
        cg = coarsen.build_coarse_graph(g, m)
        out[f"g{i}_cxadj"] = cg.xadj
        out[f"g{i}_cadj"] = cg.adj
        thr = 20 if g.num_vertices < 1000 else 100
        h = coarsen.coarsen_all(g, threshold=thr, num_workers=1)
        out[f"g{i}_thr"] = np.int64(thr)
        out[f"g{i}_depth"] = np.int64(h.depth)
        out[f"g{i}_stalled"] = np.int64(h.stalled)
        for L, (gl, ml_) in enumerate(zip(h.graphs[1:], h.mappings)):
            out[f"g{i}_L{L + 1}_xadj"] = gl.xadj
            out[f"g{i}_L{L + 1}_adj"] = gl.adj
            out[f"g{i}_M{L}_map"] = ml_.map
    out["names"] = np.asarray(names)
    save("coarsen.npz", **out)


def make_csr():
    rng = np.random.default_rng(5)
    out = {}
    k = 0
    for n, V in ((0, 3), (10, 4), (200, 30), (5000, 500)):
        pairs = rng.integers(0, V, size=(n, 2)) if n else np.zeros((0, 2), dtype=np.int64)
        for directed in (False, True):
            if n == 0:
                g = ml.from_edges(pairs, num_vertices=V, directed=directed)
            else:
                g = ml.from_edges(pairs, num_vertices=V, directed=directed)
            out[f"c{k}_pairs"] = np.asarray(pairs, dtype=np.int64)
            out[f"c{k}_V"] = np.int64(V)
            out[f"c{k}_directed"] = np.int64(directed)
            out[f"c{k}_xadj"] = g.xadj
            out[f"c{k}_adj"] = g.adj
            k += 1
    out["n"] = np.int64(k)
    save("csr.npz", **out)


def make_pool():
    out = {}
    cases = []
    k = 0
    gs = [synth.gnp_graph(40, 0.2, seed=5), synth.planted_graph(3, 10, 0.5, 0.1, seed=7),
          synth.gnp_graph(9, 0.6, seed=1)]
    pack_graphs("g", gs, out)
    for gi, g in enumerate(gs):
        n = g.num_vertices
        plan = bigtrain.PartitionPlan(K=3, boundaries=(np.arange(4, dtype=np.int64) * n) // 3)
        for pair in ((0, 0), (1, 0), (2, 1), (2, 2)):
            for d, B, n_neg, reuse in ((8, 4, 3, False), (33, 2, 1, True), (128, 3, 2, False),
                                       (8, 5, 3, True)):
                seed = 100 + k
                pool = bigtrain.build_sample_pool(g, plan, pair, B, seed)
                M = trainer.init_embedding(n, d, seed=k)
                j, kk = pair
                lo_j, hi_j = plan.part_range(j)
                lo_k, hi_k = plan.part_range(kk)
                Mj = M[lo_j:hi_j].copy()
                Mk = Mj if j == kk else M[lo_k:hi_k].copy()
                out[f"c{k}_Mj0"] = Mj.copy()
                out[f"c{k}_Mk0"] = Mk.copy()
                lr = 0.03125 + 0.01 * k
                pos = bigtrain.train_pair(Mj, Mk, pool, n_neg, lr, seed,
                                          reuse_updated_source=reuse)
                out[f"c{k}_tj"] = pool.targets_j
                if pool.targets_k is not None:
                    out[f"c{k}_tk"] = pool.targets_k
                out[f"c{k}_Mj"] = Mj
                out[f"c{k}_Mk"] = Mk
                cases.append((gi, j, kk, lo_j, hi_j, lo_k, hi_k, d, B, n_neg, int(reuse), seed,
                              lr, pos))
                k += 1
    out["cases"] = np.asarray(cases, dtype=np.float64)
    ds = [bigtrain._derived_seed(s, st, p) for s in (1, 7, 2**40) for st in (0, 3)
          for p in (0, 1, 99)]
    out["derived"] = np.asarray(ds, dtype=np.uint64)
    save("pool.npz", **out)


def make_large_and_multilevel():
    out = {}
    g = synth.planted_graph(4, 12, 0.4, 0.05, seed=6)
    pack_graphs("g", [g], out)
    runs = []
    for k, (d, e_i, B, unit, reuse) in enumerate(((8, 12, 2, "vertex-pass", False),
                                                   (16, 3, 3, "edge-scaled", False),
                                                   (8, 6, 1, "vertex-pass", True))):
        cfg = ml.TrainConfig(dim=d, total_epochs=e_i, seed=3 + k, negative_samples=2,
                             epoch_unit=unit, reuse_updated_source=reuse)
        M = trainer.init_embedding(g.num_vertices, d, seed=3 + k)
        out[f"r{k}_M0"] = M.copy()
        per_row = 3 * d * 4 + 4 * 2 * B * 4
        budget = ml.MemoryBudget(per_row * (-(-g.num_vertices // 3)) + 256, batch_size=B)
        st = bigtrain.train_large(g, M, cfg, e_i, budget, rng_stream=k)
        out[f"r{k}_M"] = M.copy()
        runs.append((d, e_i, B, 1 if unit == "edge-scaled" else 0, int(reuse), 3 + k,
                     budget.resident_bytes, st["rotations"], st["K"], st["switches"],
                     st["pos_updates"]))
    out["large"] = np.asarray(runs, dtype=np.int64)
    # multilevel end to end with the deterministic ladder
    ml_runs = []
    for k, (gname, d, e, p, unit) in enumerate((("cl", 16, 40, 0.3, "edge-scaled"),
                                                ("gnp", 8, 12, 0.5, "vertex-pass"))):
        gg = (synth.chung_lu_graph(600, 2000, 2.5, seed=8) if gname == "cl"
              else synth.gnp_graph(150, 0.05, seed=4))
        pack_graphs(f"ml{k}_", [gg], out)
        cfg = ml.TrainConfig(dim=d, total_epochs=e, smoothing_ratio=p, seed=5 + k,
                             epoch_unit=unit)
        h = coarsen.coarsen_all(gg, threshold=30, num_workers=1)
        M = trainer.train_multilevel(gg, cfg, hierarchy=h)
        out[f"ml{k}_M"] = M
        ml_runs.append((d, e, int(p * 10), 1 if unit == "edge-scaled" else 0, 5 + k, 30,
                        h.depth))
    out["multilevel"] = np.asarray(ml_runs, dtype=np.int64)
    save("large.npz", **out)


def make_rmat():
    # the reference has no R-MAT generator; pin the oracle's generator against
    # the reference CSR builder (from_edges) on its edges
    out = {}
    for k, (scale, n, seed) in enumerate(((8, 2000, 7), (10, 8000, 3))):
        perm = oracle.rmat_permutation(scale, seed)
        src, dst = oracle.rmat_edges(scale, n, seed, perm)
        g = ml.from_edges(np.column_stack([src, dst]), num_vertices=1 << scale)
        out[f"r{k}_perm"] = perm
        out[f"r{k}_src"] = src
        out[f"r{k}_dst"] = dst
        out[f"r{k}_xadj"] = g.xadj
        out[f"r{k}_adj"] = g.adj
        out[f"r{k}_cfg"] = np.asarray([scale, n, seed], dtype=np.int64)
    save("rmat.npz", **out)


def make_eval():
    # evaluate.py: midrank AUCROC with heavy ties, and train_logreg +
    # predict_scores on Hadamard features of a fixed embedding
    from mlembed import evaluate as rev
    out = {}
    rng = np.random.default_rng(11)
    for k, (n, levels) in enumerate(((50, 4), (2000, 37), (5000, 100000), (777, 1))):
        s = np.round(rng.normal(size=n) * levels) / levels
        y = (rng.random(n) < 0.4).astype(np.int8)
        y[0], y[1] = 1, 0
        out[f"a{k}_scores"] = s
        out[f"a{k}_labels"] = y
        out[f"a{k}_auc"] = np.float64(rev.auc_roc(s, y))
    g = synth.chung_lu_graph(400, 1600, 2.5, seed=9)
    M = trainer.init_embedding(g.num_vertices, 16, 3) * 40.0
    pos = g.undirected_pairs()
    neg = rev.sample_negative_edges(g, pos.shape[0], seed=5)
    pairs = np.vstack([pos, neg])
    labels = np.concatenate([np.ones(len(pos), np.int8), np.zeros(len(neg), np.int8)])
    f = rev.hadamard_features(M, pairs, labels)
    out["M"] = M
    out["pairs"] = pairs
    out["labels"] = labels
    out["rows"] = f.rows
    out["neg"] = neg
    for k, hyper in enumerate((rev.LogRegConfig(epochs=20, seed=4),
                               rev.LogRegConfig(epochs=3, batch_size=100, step=0.5, seed=2),
                               rev.LogRegConfig(seed=1, single_pass=True))):
        model = rev.train_logreg(f, hyper)
        sc = rev.predict_scores(model, f.rows)
        out[f"l{k}_hyper"] = np.asarray([hyper.epochs, hyper.batch_size, hyper.seed,
                                         int(hyper.single_pass)], dtype=np.int64)
        out[f"l{k}_step"] = np.float64(hyper.step)
        out[f"l{k}_w"] = model.weights
        out[f"l{k}_b"] = np.float64(model.bias)
        out[f"l{k}_scores"] = sc
        out[f"l{k}_auc"] = np.float64(rev.auc_roc(sc, labels))
    save("eval.npz", **out)


def _edge_text(rng, n_lines, id_pool, bad_at=None):
    """Edge-list text exercising the parser: comments (leading whitespace
    too), blank and whitespace-only lines, tabs / CR / vertical tab
    separators, signs, leading zeros, digit underscores, negative and sparse
    ids, duplicates and self-loops."""
    out = []
    for i in range(n_lines):
        r = rng.random()
        if r < 0.04:
            out.append("# comment %d" % i)
        elif r < 0.06:
            out.append("   #indented comment")
        elif r < 0.08:
            out.append(" \t ")
        else:
            u, v = (int(x) for x in rng.choice(id_pool, size=2))
            if rng.random() < 0.05:
                v = u
            fu, fv = str(u), str(v)
            k = rng.random()
            if k < 0.05 and u >= 0:
                fu = "+" + fu
            elif k < 0.1 and u >= 0:
                fu = "00" + fu
            elif k < 0.15 and len(fv) > 2 and v >= 0:
                fv = fv[0] + "_" + fv[1:]
            sep = [" ", "\t", "  ", " \x0b"][int(rng.integers(4))]
            tail = ["", " ", "\r", "\t"][int(rng.integers(4))]
            out.append(fu + sep + fv + tail)
    if bad_at is not None:
        out[bad_at[0]] = bad_at[1]
    return "\n".join(out) + "\n"


def make_edgelist():
    """load_edge_list (graph.py:134-171): parsed CSR + orig_ids of texts, and
    the exact error (type, line, message) of malformed ones."""
    import io
    from mlembed import errors as rerr
    rng = np.random.default_rng(21)
    out = {}
    pools = [np.arange(0, 50), np.concatenate([-np.arange(1, 30), 10**np.arange(3, 18)]),
             rng.integers(-2**62, 2**62, size=300)]
    k = 0
    for pool in pools:
        for directed in (False, True):
            t = _edge_text(rng, 400, pool)
            g = ml.load_edge_list(io.StringIO(t), directed=directed)
            out[f"t{k}_text"] = np.frombuffer(t.encode("ascii"), dtype=np.uint8)
            out[f"t{k}_directed"] = np.int64(directed)
            out[f"t{k}_xadj"] = g.xadj
            out[f"t{k}_adj"] = g.adj
            out[f"t{k}_orig"] = g.orig_ids
            k += 1
    out["n_text"] = np.int64(k)
    bad = ["1 2 3", "7", "x 4", "1_ 2", "1__2 3", "_1 2", "+-1 2", "0x10 3", "1.0 2",
           "5 9 # trailing comment", "\u00e91 2", "99999999999999999999 1"]
    e = 0
    for b in bad:
        for where in (3, 150):
            t = _edge_text(rng, 200, pools[0], bad_at=(where, b))
            try:
                ml.load_edge_list(io.StringIO(t))
                kind, line, msg = "none", 0, ""
            except rerr.EdgeListParseError as ex:
                kind, line, msg = "parse", ex.line_number, str(ex)
            except OverflowError as ex:
                kind, line, msg = "overflow", 0, str(ex)
            out[f"e{e}_text"] = np.frombuffer(t.encode("utf-8"), dtype=np.uint8)
            out[f"e{e}_kind"] = np.frombuffer(kind.encode(), dtype=np.uint8)
            out[f"e{e}_line"] = np.int64(line)
            out[f"e{e}_msg"] = np.frombuffer(msg.encode("utf-8"), dtype=np.uint8)
            e += 1
    out["n_err"] = np.int64(e)
    save("edgelist.npz", **out)


GENERATORS = {"rng": make_rng, "update": make_update, "train_pass": make_train_pass,
              "coarsen": make_coarsen, "csr": make_csr, "pool": make_pool,
              "large": make_large_and_multilevel, "rmat": make_rmat, "eval": make_eval,
              "edgelist": make_edgelist}

if __name__ == "__main__":
    for name in (sys.argv[1:] or GENERATORS):
        GENERATORS[name]()
