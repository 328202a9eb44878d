/*
 * gosh_b200.h -- C ABI of the B200-native GOSH multilevel-embedding path.
 *
 * This is the drop-in boundary.  The reference (mlembed, Python + numba) has
 * no FFI; its operator boundary is the set of numba kernels that take raw
 * numpy arrays and mutate them in place.  Every entry point below replaces
 * one of those kernels (cited file:line under /root/reference/pkg/src/mlembed)
 * and keeps its argument meaning.  Differences forced by the device:
 *
 *   - all array arguments are DEVICE pointers (CUDA global memory), plain
 *     C types only; the caller owns every buffer;
 *   - work that needs scratch space takes a caller-provided workspace whose
 *     size is reported by the matching *_workspace() query;
 *   - every call is asynchronous on `stream` (a cudaStream_t passed as void*),
 *     except the ones documented as "synchronizes" (they return a count that
 *     sizes the caller's next allocation);
 *   - every call returns GB_OK (0) or a negative GB_E* code; gb_last_error()
 *     returns a thread-local message for the most recent failure.
 *
 * Host binding used by the package: ctypes (paper_2008_12336_b200/_lib.py).
 */
#ifndef GOSH_B200_H
#define GOSH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GB_OK 0
#define GB_E_INVALID (-1)   /* bad argument (maps to ValueError)          */
#define GB_E_CUDA (-2)      /* CUDA runtime error (maps to RuntimeError)  */
#define GB_E_WORKSPACE (-3) /* workspace too small                        */
#define GB_E_UNSUPPORTED (-4)

/* train flags */
#define GB_TRAIN_REUSE 1u  /* TrainConfig.reuse_updated_source (trainer.py:47-50) */
#define GB_TRAIN_EXACT 2u  /* one source group, reference order, serial fp64 dot  */
#define GB_TRAIN_FAST_SIGMOID 4u /* non-exact: fp32 cancellation-free sigmoid     */
#define GB_TRAIN_ATOMIC 8u /* non-exact: sample rows written back by vector reductions (no lost updates) */

/* csr build flags */
#define GB_CSR_DROP_SELF 1u  /* from_edges drops self-loops (graph.py:127-128)  */
#define GB_CSR_SYMMETRIZE 2u /* undirected: add reversed arcs (graph.py:129-130) */

/* status block written by the training kernels (device memory, 4 x int64):
 *   [0] non-finite flag (0/1)            -- fused replacement of the
 *   [1] first epoch that saw a non-finite    isfinite scan, trainer.py:236-237
 *   [2] positive updates applied (pool kernels; train_pair return value)
 *   [3] negative updates applied (pool kernels)                               */
#define GB_STATUS_WORDS 4

const char *gb_last_error(void);
int gb_version(void);
/* Device properties the host planner needs (SM count, max resident warps). */
int gb_device_info(int device, int *num_sms, int *max_warps_per_sm);

/* ---- L0: counter-based RNG (_rng.py:19-49) -------------------------------
 * out[i] = draw_below(stream_key(seed, stream, step, vertex0 + i), counter, n)
 * Used by tests to pin the device RNG against the reference bit-for-bit. */
int gb_rng_draw_below(uint64_t seed, uint64_t stream, uint64_t step,
                      uint64_t vertex0, uint64_t counter, int64_t n,
                      int64_t count, int64_t *out, void *stream_handle);

/* ---- L1: CSR build (graph.py:93-131 _csr_from_arcs / from_edges) ---------
 * Builds xadj[V+1] (int64) and adj[cap] (int32) from parallel arc arrays.
 * adj must hold 2*num_arcs entries when GB_CSR_SYMMETRIZE is set, else
 * num_arcs.  Rows come out strictly ascending and deduplicated.  Synchronizes
 * and writes the number of stored arcs to *num_edges_out (host pointer). */
int gb_csr_build_workspace(int64_t num_vertices, int64_t num_arcs,
                           unsigned flags, size_t *bytes);
int gb_csr_build(int64_t num_vertices, const int64_t *src, const int64_t *dst,
                 int64_t num_arcs, unsigned flags, int64_t *xadj, int32_t *adj,
                 int64_t *num_edges_out, void *workspace, size_t ws_bytes,
                 void *stream_handle);

/* Row-block ("chunked") CSR construction, for graphs whose one-shot key
 * buffers (24 B per arc) exceed the device (C5: ~8B arcs).  Same result as
 * gb_csr_build / gb_coarse_csr, bit for bit, block by block:
 *   gb_arc_histogram     hist[s] += arcs with source s (int64[V], caller
 *                        zeroes; self-loops dropped / reversed arcs added
 *                        per flags) -- the host picks row blocks from it;
 *   gb_arc_keys_range    append key (s - r0) * V + d of every arc with
 *                        r0 <= s < r1 at keys[*cursor..] (device cursor);
 *   gb_mapped_histogram / gb_mapped_keys_range
 *                        the same for the coarse arcs (cmap[v], cmap[u]) of
 *                        a CSR with intra-cluster arcs dropped
 *                        (coarsen.py:200-253), by coarse row block;
 *   gb_keys_to_rows      sort + deduplicate a block's keys and write its
 *                        rows: xadj_rows[0..rows) offset by `base` and
 *                        adj_out[0..unique); synchronizes, *num_unique_out
 *                        is a host pointer.
 * gb_rmat_edges_range generates R-MAT samples first .. first+count-1 (each a
 * pure function of its index), so sample batches never coexist. */
int gb_arc_histogram(const int64_t *src, const int64_t *dst, int64_t num_arcs,
                     unsigned flags, int64_t *hist, void *stream_handle);
int gb_arc_keys_range(const int64_t *src, const int64_t *dst, int64_t num_arcs,
                      unsigned flags, int64_t num_vertices, int64_t r0, int64_t r1,
                      uint64_t *keys, int64_t *cursor, void *stream_handle);
int gb_mapped_histogram(const int64_t *xadj, const int32_t *adj, int64_t num_vertices,
                        const int32_t *cmap, int64_t *hist, void *stream_handle);
int gb_mapped_keys_range(const int64_t *xadj, const int32_t *adj, int64_t num_vertices,
                         const int32_t *cmap, int64_t num_clusters, int64_t c0,
                         int64_t c1, uint64_t *keys, int64_t *cursor, void *stream_handle);
/* gb_mapped_keys_rows: the keys of gb_mapped_keys_range for clusters
 * [c0, c1), appended per row instead of at one cursor: row_cursor[r]
 * (int64[c1 - c0]) holds row c0 + r's start in keys on entry (an exclusive
 * scan of gb_mapped_histogram over the block) and its end on return.  Same
 * keys, spread over per-row atomics; replaces the single-cursor form in
 * build_coarse_graph's blocks (reference coarsen.py:256-281).  heavy
 * (int64[1 + heavy_cap], or NULL with heavy_cap 0) queues the vertices of
 * more than heavy_arcs (>= 32) arcs, whose arcs are then split over all
 * warps; a full queue falls back to one warp per vertex (heavy_cap >=
 * E / heavy_arcs never fills). */
int gb_mapped_keys_rows(const int64_t *xadj, const int32_t *adj, int64_t num_vertices,
                        const int32_t *cmap, int64_t num_clusters, int64_t c0, int64_t c1,
                        int64_t *row_cursor, uint64_t *keys, int64_t *heavy,
                        int64_t heavy_cap, int64_t heavy_arcs, void *stream_handle);
int gb_keys_to_rows_workspace(int64_t num_keys, int64_t rows, int64_t num_cols,
                              size_t *bytes);
int gb_keys_to_rows(uint64_t *keys, int64_t num_keys, int64_t rows, int64_t num_cols,
                    int64_t base, int64_t *xadj_rows, int32_t *adj_out,
                    int64_t *num_unique_out, void *workspace, size_t ws_bytes,
                    void *stream_handle);
int gb_rmat_edges_range(int scale, int64_t first, int64_t count, double t_a, double t_ab,
                        double t_abc, uint64_t seed, const int64_t *perm, int64_t *src,
                        int64_t *dst, void *stream_handle);

/* Drop isolated vertices and re-densify ids in ascending order -- the
 * load_edge_list convention (graph.py:160-164) applied to a CSR.  new_id
 * receives the old->new map (-1 for dropped ids); kept receives new->old.
 * Synchronizes; writes the kept-vertex count to *num_kept_out. */
int gb_csr_densify_workspace(int64_t num_vertices, size_t *bytes);
int gb_csr_densify(int64_t num_vertices, int64_t num_edges,
                   const int64_t *xadj, const int32_t *adj, int64_t *xadj_out,
                   int32_t *adj_out, int64_t *new_id, int64_t *kept,
                   int64_t *num_kept_out, void *workspace, size_t ws_bytes,
                   void *stream_handle);

/* Non-isolated vertices in ascending id order (the sources a training pass
 * visits, trainer.py:198-200).  Synchronizes; writes the count. */
int gb_active_sources_workspace(int64_t num_vertices, size_t *bytes);
int gb_active_sources(int64_t num_vertices, const int64_t *xadj, int32_t *out,
                      int64_t *count_out, void *workspace, size_t ws_bytes,
                      void *stream_handle);

/* ---- synthetic input: Graph500 R-MAT edge sampler -------
 * Writes num_samples (src,dst) pairs over 2^scale ids; ids are relabelled by
 * the seeded permutation perm (perm[i] = i-th id of the stable argsort of
 * mix-keys, computed by gb_rmat_permutation).  thresholds = {a, a+b, a+b+c}. */
int gb_rmat_permutation_workspace(int scale, size_t *bytes);
int gb_rmat_permutation(int scale, uint64_t seed, int64_t *perm,
                        void *workspace, size_t ws_bytes, void *stream_handle);
int gb_rmat_edges(int scale, int64_t num_samples, double t_a, double t_ab,
                  double t_abc, uint64_t seed, const int64_t *perm,
                  int64_t *src, int64_t *dst, void *stream_handle);

/* ---- L2: coarsening (coarsen.py) ------------------------------------------
 * degree_order: order[V] by (-deg, +id)   (coarsen.py:69-95 _counting_order) */
int gb_degree_order_workspace(int64_t num_vertices, size_t *bytes);
int gb_degree_order(int64_t num_vertices, const int64_t *xadj, int64_t *order,
                    void *workspace, size_t ws_bytes, void *stream_handle);

/* collapse: cluster map identical to _collapse_seq (coarsen.py:98-114) for
 * the given order; delta = num_edges/num_vertices as the reference computes
 * it (coarsen.py:161).  Order-priority rounds, bit-exact by construction
 * (SURVEY.md Appendix B).  xadj gives the (out-)degrees; in_xadj/in_adj is
 * the in-arc CSR (the same arrays for an undirected graph, the transpose
 * for a directed one).  Synchronizes; writes the cluster count. */
int gb_collapse_workspace(int64_t num_vertices, size_t *bytes);
int gb_collapse(int64_t num_vertices, const int64_t *xadj, const int64_t *in_xadj,
                const int32_t *in_adj, const int64_t *order, double delta, int32_t *cmap,
                int64_t *num_clusters_out, int *rounds_out, void *workspace,
                size_t ws_bytes, void *stream_handle);

/* run-dependent parallel collapse: the reference's try-lock mode
 * (coarsen.py:117-179 _collapse_par + _normalize; collapse_map_parallel).
 * num_workers warps grab GRAB_BATCH=64 order positions at a time, claim hubs
 * and members with CAS and skip on a lost race; hubs are renumbered by order
 * position.  num_workers=1 equals gb_collapse; more workers give a valid,
 * interleaving-dependent map (not in the parity contract, coarsen.py:11-13).
 * xadj/adj is the out-arc CSR, as in the reference.  Synchronizes. */
int gb_collapse_cas_workspace(int64_t num_vertices, size_t *bytes);
int gb_collapse_cas(int64_t num_vertices, const int64_t *xadj, const int32_t *adj,
                    const int64_t *order, double delta, int64_t num_workers, int32_t *cmap,
                    int64_t *num_clusters_out, void *workspace, size_t ws_bytes,
                    void *stream_handle);

/* coarse CSR: row c = sorted unique {map[u] : u in N(members of c)} \ {c}
 * (coarsen.py:182-281 build_coarse_graph).  adj_out must hold num_edges
 * entries.  Synchronizes; writes the coarse arc count. */
int gb_coarse_csr_workspace(int64_t num_vertices, int64_t num_edges,
                            int64_t num_clusters, size_t *bytes);
int gb_coarse_csr(int64_t num_vertices, int64_t num_edges, const int64_t *xadj,
                  const int32_t *adj, const int32_t *cmap, int64_t num_clusters,
                  int64_t *xadj_out, int32_t *adj_out, int64_t *num_edges_out,
                  void *workspace, size_t ws_bytes, void *stream_handle);

/* ---- L3: projection (trainer.py:243-249 expand_embedding) ----------------
 * out[v, :] = coarse[cmap[v], :] for v < num_rows. */
/* Position-keyed checksum of an int32 / int64 device array (elem_bytes 4 or
 * 8): *out = sum_i mix64((i * 0x9E3779B97F4A7C15) ^ (uint64)(int64)x[i])
 * mod 2^64 (out is a device uint64).  Not a reference kernel: the parity
 * check for hierarchies too large to ship as fixtures (tests compare it with
 * the oracle's or_checksum of the reference's arrays). */
int gb_checksum(const void *data, int64_t n, int elem_bytes, uint64_t *out,
                void *stream_handle);

int gb_expand(const float *coarse, int64_t num_clusters, int dim,
              const int32_t *cmap, int64_t num_rows, float *out,
              void *stream_handle);

/* ---- L3: VERSE/NCE training passes (trainer.py:184-207 _train_pass) ------
 * Runs passes pass_begin .. pass_begin+n_passes-1 of one level.  Pass p uses
 * learning rate lr_per_epoch[p / passes_per_epoch] (float32 values, as
 * train_level computes them, trainer.py:230) and RNG step p.  Sources are
 * owned by "groups" (G lanes of a warp); max_groups caps how many sources are
 * in flight at once (0 = fill the GPU).  GB_TRAIN_EXACT runs one group in
 * the reference's sequential order with the reference's serial fp64 dot and
 * reproduces _train_pass(num_workers=1) bit-for-bit.  sources (optional,
 * from gb_active_sources) lists the non-isolated vertices in ascending order
 * so lanes never idle on isolated ids; NULL scans all V.  status: above. */
int gb_train_passes(int64_t num_vertices, const int64_t *xadj,
                    const int32_t *adj, const int32_t *sources,
                    int64_t n_sources, float *M, int dim, int n_neg,
                    uint64_t seed, uint64_t rng_stream, int64_t pass_begin,
                    int64_t n_passes, int64_t passes_per_epoch,
                    const float *lr_per_epoch, unsigned flags,
                    int64_t max_groups, int64_t *status, void *stream_handle);

/* gb_train_passes with positives from VERSE's personalized-PageRank
 * similarity instead of the reference's adjacency similarity (SURVEY.md 8(f)
 * rank 4; not in the reference): a walk from v that continues to
 * a uniform neighbour while a uniform draw is below ppr_alpha (0 < alpha < 1;
 * VERSE uses 0.85), capped at 64 steps; the sample is the vertex reached (v
 * itself with probability 1 - alpha).  alpha is used rounded to float32.
 * Negatives, update rule, EXACT mode and status are those of
 * gb_train_passes. */
int gb_train_passes_ppr(int64_t num_vertices, const int64_t *xadj, const int32_t *adj,
                        const int32_t *sources, int64_t n_sources, float *M, int dim, int n_neg,
                        uint64_t seed, uint64_t rng_stream, int64_t pass_begin, int64_t n_passes,
                        int64_t passes_per_epoch, const float *lr_per_epoch, unsigned flags,
                        int64_t max_groups, int64_t *status, double ppr_alpha,
                        void *stream_handle);

/* Fixed sample lists (update_embedding, trainer.py:137-142, generalized):
 * source src[i] is updated against samples[i*k + j] for j = 0..k-1 in order
 * (-1 skips a slot) with label labels[j] (1 positive, 0 negative), single-
 * array semantics, lr as float64.  Different sources run concurrently
 * (Hogwild) unless GB_TRAIN_EXACT, which applies the lists in index order. */
int gb_apply_sample_lists(float *M, int dim, int64_t n_src, const int64_t *src,
                          int k, const int64_t *samples, const int8_t *labels,
                          double lr, unsigned flags, int64_t max_groups,
                          int64_t *status, void *stream_handle);

/* Full-matrix non-finite scan (fallback half of trainer.py:236-237; rows no
 * update touched).  Sets status[0] and status[1]=epoch when any entry is
 * NaN/Inf. */
int gb_nonfinite_scan(const float *M, int64_t count, int64_t epoch,
                      int64_t *status, void *stream_handle);

/* ---- L3b: partitioned trainer (bigtrain.py) --------------------------------
 * _fill_pool_side (bigtrain.py:164-196): out[(v-lo_s)*B + t] for v in
 * [lo_s, hi_s): B uniform draws from N(v) & [lo_t, hi_t), -1 if empty. */
int gb_fill_pool_side(const int64_t *xadj, const int32_t *adj, int64_t lo_s,
                      int64_t hi_s, int64_t lo_t, int64_t hi_t, int B,
                      uint64_t seed, uint64_t side, int32_t *out,
                      void *stream_handle);

/* _train_pool_side (bigtrain.py:215-238): sources i < n_src of Msrc, B
 * pooled targets each (global ids, minus lo_t), n_neg negatives drawn from
 * [0, n_t) with key(seed, side, 1, i).  lr is float64 as in train_large
 * (bigtrain.py:432).  When Msrc == Mtgt (diagonal pair) a self-sample uses
 * the load-once rule of the reference's noalias kernel.
 * If targets == NULL the pool is drawn on the fly from the device CSR
 * (xadj/adj, source ids lo_s + i, pool side pool_side, pool key
 * key(seed, pool_side, 0, v)) -- bit-identical to a materialized pool.
 * status[2] += positive updates applied. */
int gb_train_pool_side(float *Msrc, float *Mtgt, int dim,
                       const int32_t *targets, int64_t n_src, int B,
                       int64_t lo_t, int64_t n_t, int n_neg, double lr,
                       uint64_t seed, uint64_t side, const int64_t *xadj,
                       const int32_t *adj, int64_t lo_s, uint64_t pool_side,
                       unsigned flags, int64_t max_groups, int64_t *status,
                       void *stream_handle);

/* Compacted pool side for the pair kernel (same draws as gb_fill_pool_side):
 * sources v in [lo_s, hi_s) with at least one neighbour in [lo_t, hi_t) get
 * an entry k < *count: list[k] = v - lo_s, targets[k*B + t] = pool slot t
 * (global id).  Sources without one train nothing in _train_pool_side
 * (bigtrain.py:229-231) and are left out.  Entry order is id order within a
 * warp of 32 sources, warps in any order.  list holds hi_s-lo_s entries,
 * targets (hi_s-lo_s)*B; count is a device int64 (set by this call). */
int gb_fill_pool_compact(const int64_t *xadj, const int32_t *adj, int64_t lo_s,
                         int64_t hi_s, int64_t lo_t, int64_t hi_t, int B,
                         uint64_t seed, uint64_t side, int32_t *list,
                         int32_t *targets, int64_t *count, void *stream_handle);

/* _train_pool_side over a compacted pool (gb_fill_pool_compact): entry
 * k < min(max_src, *count) trains local source list[k] against
 * targets[k*B ..]; everything else as gb_train_pool_side (negatives keyed by
 * the source's local id, so results equal the uncompacted launch up to the
 * order sources run in). */
int gb_train_pool_list(float *Msrc, float *Mtgt, int dim, const int32_t *list,
                       const int32_t *targets, const int64_t *count,
                       int64_t max_src, int B, int64_t lo_t, int64_t n_t,
                       int n_neg, double lr, uint64_t seed, uint64_t side,
                       unsigned flags, int64_t max_groups, int64_t *status,
                       void *stream_handle);

/* Balanced pools (an opt-in alternative to the reference's fixed-B pools,
 * not in the reference): every source v in [lo_s, hi_s) with deg(v) > 0 gets
 * an entry k < *count with list[k] = v - lo_s, first[k]/cnt[k] = its
 * neighbours in [lo_t, hi_t) as a range of adj, and npos[k] =
 * floor(BK*cnt/deg + u) positives (u uniform from key(seed, side, 2, v)):
 * over a rotation of K parts with BK = B*K the positives follow the
 * in-memory pass's neighbour distribution in expectation. */
int gb_fill_pool_balanced(const int64_t *xadj, const int32_t *adj, int64_t lo_s,
                          int64_t hi_s, int64_t lo_t, int64_t hi_t, int64_t BK,
                          uint64_t seed, uint64_t side, int32_t *list,
                          int64_t *first, int32_t *cnt, int32_t *npos,
                          int64_t *count, void *stream_handle);

/* Pair side over balanced pools: entry k trains local source list[k] with
 * B slots (slot t: a positive iff t < npos[k], then n_neg negatives from
 * key(seed, side, 1, i)), then npos[k] - B further positives if npos[k] > B;
 * positive t = adj[first[k] + draw_below(key(seed, pool_side, 0, lo_s + i),
 * t, cnt[k])] - lo_t.  Otherwise as gb_train_pool_list. */
int gb_train_pool_balanced(float *Msrc, float *Mtgt, int dim, const int32_t *list,
                           const int64_t *first, const int32_t *cnt,
                           const int32_t *npos, const int64_t *count,
                           int64_t max_src, int B, int64_t lo_t, int64_t n_t,
                           int n_neg, double lr, uint64_t seed, uint64_t side,
                           const int32_t *adj, int64_t lo_s, uint64_t pool_side,
                           unsigned flags, int64_t max_groups, int64_t *status,
                           void *stream_handle);

/* Page-lock a caller host buffer in place (cudaHostRegister) so part
 * switches of the partitioned trainer DMA straight from / into the caller's
 * embedding matrix (bigtrain.py:275-299 host staging) without a pinned copy. */
int gb_host_register(void *ptr, size_t bytes);
int gb_host_unregister(void *ptr);

/* ---- L5: split and negative pairs (graph.py:46-59, 222-265;
 * evaluate.py:80-125), SURVEY.md 8(f) rank 3.  The random choices stay
 * numpy's (host); these do the O(|E|) work around them.
 * undirected_pairs: arcs (u, v) with u < v in CSR order into pu/pv
 * (capacity entries); *num_pairs set (synchronizes the stream). */
int gb_undirected_pairs_workspace(int64_t num_vertices, size_t *bytes);
int gb_undirected_pairs(const int64_t *xadj, const int32_t *adj,
                        int64_t num_vertices, int64_t *pu, int64_t *pv,
                        int64_t capacity, int64_t *num_pairs, void *workspace,
                        size_t workspace_bytes, void *stream_handle);

/* split_train_test's partition: pairs chosen[k] (indices into pu/pv) are
 * withheld; vertices touched by the remaining pairs are kept and relabelled
 * densely in ascending order (relabel[V]: new id or -1; kept[]: old ids);
 * train pairs (relabelled) and the test pairs whose endpoints both survive
 * (relabelled) are compacted in pair order.  counts (host) = {train pairs,
 * test pairs, kept vertices}; synchronizes the stream. */
int gb_split_partition_workspace(int64_t num_pairs, int64_t num_vertices,
                                 size_t *bytes);
int gb_split_partition(const int64_t *pu, const int64_t *pv, int64_t num_pairs,
                       const int64_t *chosen, int64_t k, int64_t num_vertices,
                       int64_t *train_u, int64_t *train_v, int64_t *test_u,
                       int64_t *test_v, int64_t *relabel, int64_t *kept,
                       int64_t *counts, void *workspace, size_t workspace_bytes,
                       void *stream_handle);

/* out[i] = 1 iff (u[i], v[i]) is an arc or (u, v) / (v, u) is one of the
 * excluded pairs -- sample_negative_edges' rejection test. */
int gb_pairs_member_workspace(int64_t num_excluded, size_t *bytes);
int gb_pairs_member(const int64_t *xadj, const int32_t *adj, int64_t num_vertices,
                    const int64_t *u, const int64_t *v, int64_t n,
                    const int64_t *excl_u, const int64_t *excl_v,
                    int64_t num_excluded, uint8_t *out, void *workspace,
                    size_t workspace_bytes, void *stream_handle);

/* ---- L4: link-prediction evaluator (evaluate.py), SURVEY.md 8(f) rank 1 ----
 * hadamard_features (evaluate.py:69-78): X[i*dim+t] = fl32(M[u_i,t]*M[v_i,t])
 * for pairs[2i]=u_i, pairs[2i+1]=v_i. */
int gb_hadamard_features(const float *M, int64_t num_rows, int dim,
                         const int64_t *pairs, int64_t n, float *X,
                         void *stream_handle);

/* One epoch of train_logreg's mini-batch descent (evaluate.py:128-140) over
 * the permutation perm[n] (numpy's rng.permutation, drawn on the host):
 * batches of batch_size rows in perm order, w (dim doubles) and *b updated
 * in place in device memory. */
int gb_logreg_epoch(const float *X, int dim, const int8_t *labels,
                    const int64_t *perm, int64_t n, int batch_size,
                    double step, double *w, double *b, void *stream_handle);

/* predict_scores (evaluate.py:146-147): out[i] = X[i] . w + b (fp64). */
int gb_predict_scores(const float *X, int dim, int64_t n, const double *w,
                      double b, double *out, void *stream_handle);

/* auc_roc (evaluate.py:150-167): *rank2_pos (device) = sum over positives
 * of doubled midranks; AUC = (r2p - P(P+1)) / (2 P N) on the host. */
int gb_auc_roc_workspace(int64_t n, size_t *bytes);
int gb_auc_roc(const double *scores, const int8_t *labels, int64_t n,
               unsigned long long *rank2_pos, void *workspace,
               size_t workspace_bytes, void *stream_handle);

/* ---- device-parameter forms for CUDA-graph replay -------------------------
 * gb_fill_pool_side / gb_train_pool_side / gb_fill_pool_compact /
 * gb_train_pool_list / gb_fill_pool_balanced / gb_train_pool_balanced with the pair's seed and lr read at run time from
 * `param`, a device pointer to {uint64 seed; double lr;} (16 bytes), instead
 * of the scalar arguments.  A rotation of the part-pair tournament is the
 * same launch sequence every time except for these two values, so it is
 * captured once into a CUDA graph and replayed with a rewritten parameter
 * table (tournament.py).  Results equal the scalar forms. */
int gb_fill_pool_side_dp(const int64_t *xadj, const int32_t *adj, int64_t lo_s, int64_t hi_s,
                         int64_t lo_t, int64_t hi_t, int B, const void *param, uint64_t side,
                         int32_t *out, void *stream_handle);
int gb_train_pool_side_dp(float *Msrc, float *Mtgt, int dim, const int32_t *targets,
                          int64_t n_src, int B, int64_t lo_t, int64_t n_t, int n_neg,
                          const void *param, uint64_t side, const int64_t *xadj,
                          const int32_t *adj, int64_t lo_s, uint64_t pool_side, unsigned flags,
                          int64_t max_groups, int64_t *status, void *stream_handle);
int gb_fill_pool_compact_dp(const int64_t *xadj, const int32_t *adj, int64_t lo_s,
                            int64_t hi_s, int64_t lo_t, int64_t hi_t, int B, const void *param,
                            uint64_t side, int32_t *list, int32_t *targets, int64_t *count,
                            void *stream_handle);
int gb_train_pool_list_dp(float *Msrc, float *Mtgt, int dim, const int32_t *list,
                          const int32_t *targets, const int64_t *count, int64_t max_src, int B,
                          int64_t lo_t, int64_t n_t, int n_neg, const void *param, uint64_t side,
                          unsigned flags, int64_t max_groups, int64_t *status,
                          void *stream_handle);
int gb_fill_pool_balanced_dp(const int64_t *xadj, const int32_t *adj, int64_t lo_s,
                             int64_t hi_s, int64_t lo_t, int64_t hi_t, int64_t BK,
                             const void *param, uint64_t side, int32_t *list, int64_t *first,
                             int32_t *cnt, int32_t *npos, int64_t *count, void *stream_handle);
int gb_train_pool_balanced_dp(float *Msrc, float *Mtgt, int dim, const int32_t *list,
                              const int64_t *first, const int32_t *cnt, const int32_t *npos,
                              const int64_t *count, int64_t max_src, int B, int64_t lo_t,
                              int64_t n_t, int n_neg, const void *param, uint64_t side,
                              const int32_t *adj, int64_t lo_s, uint64_t pool_side,
                              unsigned flags, int64_t max_groups, int64_t *status,
                              void *stream_handle);

/* ---- graph input on the device --------------------
 * CSR validation of a loaded GSHG file (graph.py:61-77 Graph.validate, run by
 * load_graph, graph.py:203-219).  *flags_out (host) gets a bit per failed
 * check, in the reference's order: 1 xadj endpoints, 2 xadj decreasing, 4 adj
 * entry out of range, 8 a row not strictly ascending (meaningful only when 1
 * and 2 are clear).  Synchronizes. */
int gb_csr_validate_workspace(int64_t num_edges, size_t *bytes);
int gb_csr_validate(int64_t num_vertices, int64_t num_edges, const int64_t *xadj,
                    const int32_t *adj, int *flags_out, void *workspace, size_t ws_bytes,
                    void *stream_handle);

/* Edge-list text (graph.py:134-157 load_edge_list's loop) in device memory:
 * lines end at '\n'; blank and '#' lines are skipped; a line must hold two
 * fields that Python's int() accepts ([+-]?digits with single underscores
 * between digits).  u_out/v_out (room for num_bytes/2+1 entries) receive the
 * ids of the edge lines in order.  result (host, 5 x int64): edges, lines,
 * index of the first malformed line (-1 if none), 1 if a syntactically valid
 * id lies outside int64 (the reference's later OverflowError), 1 if the text
 * holds a byte >= 0x80 or a '\r' not followed by '\n' -- text whose lines
 * or fields Python splits differently, which the caller hands to the host
 * parser (the other results are then not meaningful).  Synchronizes. */
int gb_parse_edge_text_workspace(int64_t num_bytes, size_t *bytes);
int gb_parse_edge_text(const char *text, int64_t num_bytes, int64_t *u_out, int64_t *v_out,
                       int64_t *result, void *workspace, size_t ws_bytes,
                       void *stream_handle);

/* Id densification (graph.py:160-164: np.unique, then np.searchsorted):
 * uniq (n entries of room) gets the sorted distinct values of ids; with
 * relabel, ids[i] becomes its rank in uniq.  Synchronizes. */
int gb_unique_ids_workspace(int64_t n, size_t *bytes);
int gb_unique_ids(int64_t *ids, int64_t n, int64_t *uniq, int64_t *num_unique_out,
                  int relabel, void *workspace, size_t ws_bytes, void *stream_handle);

#ifdef __cplusplus
}
#endif
#endif /* GOSH_B200_H */
