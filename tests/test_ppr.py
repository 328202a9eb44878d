"""Personalized-PageRank positives (not in the
reference, SPEC.md:14 -- VERSE's published sampler).

CPU: the oracle's restatement of the walk (gosh_oracle.c ppr_positive)
against the exact PPR distribution of a small graph -- (1-a) sum_t a^t e_v P^t,
computed by power iteration -- and config validation.  GPU: the EXACT kernel
with PPR positives bit-exact against the oracle's sequential pass; the
Hogwild kernel; the part-pair paths reject it.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2008_12336_b200 as gb
from paper_2008_12336_b200.graph import Graph


def _exact_ppr(x, a, v, alpha, steps=64):
    V = len(x) - 1
    P = np.zeros((V, V))
    for u in range(V):
        d = x[u + 1] - x[u]
        if d == 0:
            P[u, u] = 1.0  # sink: the walk stops here
        for e in range(x[u], x[u + 1]):
            P[u, a[e]] += 1.0 / d
    p = np.zeros(V)
    p[v] = 1.0
    out = np.zeros(V)
    for t in range(steps):
        out += (1 - alpha) * alpha ** t * p
        p = p @ P
    return out + alpha ** steps * p  # walks cut at the step cap


@pytest.mark.parametrize("alpha", [0.85, 0.5])
def test_oracle_walk_follows_the_ppr_distribution(orc, alpha):
    x, a = orc.rmat_graph(7, 600, 3, densify_ids=True)
    for v in (0, 5, 17):
        want = _exact_ppr(x, a, v, alpha)
        draws = orc.ppr_positives(x, a, v, alpha, 1, 0, 200_000)
        got = np.bincount(draws, minlength=len(x) - 1) / draws.shape[0]
        assert 0.5 * np.abs(got - want).sum() < 0.01  # total variation


def test_similarity_config_validation():
    with pytest.raises(gb.ConfigError):
        gb.TrainConfig(similarity="simrank").validate()
    with pytest.raises(gb.ConfigError):
        gb.TrainConfig(similarity="ppr", ppr_alpha=1.0).validate()
    gb.TrainConfig(similarity="ppr", ppr_alpha=0.85).validate()


@pytest.mark.gpu
@pytest.mark.parametrize("d,alpha", [(16, 0.85), (32, 0.5), (128, 0.85)])
def test_exact_ppr_pass_bit_exact_against_oracle(cuda, orc, d, alpha):
    x, a = orc.rmat_graph(10, 6000, 4, densify_ids=True)
    g = Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
    M0 = orc.init_embedding(g.num_vertices, d, 2)
    ref = M0.copy()
    orc.train_level(x, a, ref, d, 3, 0.035, 3, 1, 0, ppr_alpha=alpha)
    M = M0.copy()
    cfg = gb.TrainConfig(dim=d, deterministic=True, similarity="ppr", ppr_alpha=alpha)
    gb.train_level(g, M, cfg, 3)
    assert np.array_equal(M, ref)
    plain = M0.copy()
    gb.train_level(g, plain, gb.TrainConfig(dim=d, deterministic=True), 3)
    assert not np.array_equal(plain, M)  # the positives really changed


@pytest.mark.gpu
def test_hogwild_ppr_and_part_pair_rejection(cuda, orc):
    import torch
    g = gb.rmat_graph(14, 1 << 18, 7, densify_ids=True)
    cfg = gb.TrainConfig(dim=128, similarity="ppr")
    M = torch.from_numpy(orc.init_embedding(g.num_vertices, 128, 1)).cuda()
    st = gb.train_level(g, M, cfg, 2)
    assert st.updates > 0 and bool(torch.isfinite(M).all())
    with pytest.raises(gb.ConfigError):
        gb.train_tournament(g, M, cfg, 1, num_ranks=2)


@pytest.mark.gpu
@pytest.mark.parametrize("d", [32, 128])
def test_hot_ppr_pass_single_group_matches_sequential(cuda, orc, monkeypatch, d):
    """The staged HOT pass with PPR positives (fp64 sigmoid), one source in
    flight, is the oracle's sequential PPR pass up to the tree dot."""
    monkeypatch.setenv("GB_PASS_SMEM", "1")
    x, a = orc.rmat_graph(10, 6000, 4, densify_ids=True)
    g = Graph(len(x) - 1, int(x[-1]), xadj=x, adj=a)
    M0 = orc.init_embedding(g.num_vertices, d, 2) * 20.0
    ref = M0.copy()
    orc.train_level(x, a, ref, d, 2, 0.035, 3, 1, 0, ppr_alpha=0.85)
    M = M0.copy()
    gb.train_level(g, M, gb.TrainConfig(dim=d, similarity="ppr", max_inflight=1), 2)
    err = np.abs(M - ref).max() / np.abs(ref).max()
    assert err <= 1e-5, err
