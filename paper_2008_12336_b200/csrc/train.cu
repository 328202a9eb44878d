// C ABI of the training kernels: layout dispatch, grid sizing, launch.
// Kernels live in train_kernels.cuh; instantiations in train_{vec_*,scalar}.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "train_kernels.cuh"

namespace gb {
namespace tk {

Variant vec_variant_a(int G, int NV);
Variant vec_variant_b(int G, int NV);
Variant vec_variant_c(int G, int NV);

Variant vec_variant(int G, int NV) {
  Variant v = vec_variant_a(G, NV);
  if (!v.G) v = vec_variant_b(G, NV);
  if (!v.G) v = vec_variant_c(G, NV);
  return v;
}

namespace {

__global__ void nonfinite_scan_kernel(const float *__restrict__ M, int64_t n, int64_t epoch,
                                      int64_t *status) {
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(M[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) {
    atomicOr(reinterpret_cast<unsigned long long *>(status), 1ull);
    atomicMin(reinterpret_cast<long long *>(status + 1), (long long)epoch);
  }
}

// Lanes per source for a vector layout.  Throughput launches: few lanes per
// source (8 at d=128) so per-source scalar work is shared by 4 sources per
// warp.  Latency launches (capped, small levels): as many lanes as the row
// has float4s (up to 32), so the per-lane chain is shortest.  GB_GROUP_LANES
// overrides both (tuning knob; only the tree-dot summation order changes).
int preferred_lanes(int dim, bool latency) {
  const char *env = std::getenv("GB_GROUP_LANES");
  if (env) {
    int g = std::atoi(env);
    if (g == 2 || g == 4 || g == 8 || g == 16 || g == 32) return g;
  }
  if (latency) return std::max(2, std::min(32, dim / 4));
  if (dim <= 16) return std::max(dim / 4, 2);
  if (dim <= 128) return 8;
  return 16;
}

bool pick_vector(int dim, int G, Variant &out) {
  if (dim % 4 != 0 || G < 2) return false;
  const int nv4 = dim / 4;
  if (nv4 % G != 0) return false;
  out = vec_variant(G, nv4 / G);
  return out.G != 0;
}

bool pick_variant(int dim, bool aligned, bool exact, Variant &out, bool latency = false) {
  if (aligned && !exact) {
    const int G = preferred_lanes(dim, latency);
    for (int g = G; g <= 32; g *= 2)
      if (pick_vector(dim, g, out)) return true;
    for (int g = G / 2; g >= 2; g /= 2)
      if (pick_vector(dim, g, out)) return true;
  }
  const int ns = (dim + 31) / 32;
  for (int s = 1; s <= 16; s *= 2)
    if (ns <= s) {
      out = scalar_variant(s, exact);
      return out.G != 0;
    }
  return false;
}

// The default non-deterministic flags (fast sigmoid, vector-reduction
// write-back, no reuse) run the HOT instantiations when the layout has them.
// GB_NO_HOT=1 forces the run-time-flag kernels (A/B measurements).
bool use_hot(unsigned flags) {
  static const bool off = [] {
    const char *e = std::getenv("GB_NO_HOT");
    return e && std::atoi(e) != 0;
  }();
  return !off && !(flags & GB_TRAIN_EXACT) && (flags & GB_TRAIN_FAST_SIGMOID) &&
         (flags & GB_TRAIN_ATOMIC) && !(flags & GB_TRAIN_REUSE);
}

// The default flags except the fast sigmoid: the fp64-sigmoid KIND 3 pass.
bool use_hot_f64(unsigned flags) {
  static const bool off = [] {
    const char *e = std::getenv("GB_NO_HOT");
    return e && std::atoi(e) != 0;
  }();
  return !off && !(flags & GB_TRAIN_EXACT) && !(flags & GB_TRAIN_FAST_SIGMOID) &&
         (flags & GB_TRAIN_ATOMIC) && !(flags & GB_TRAIN_REUSE);
}

void select_hot(Variant &v, unsigned flags, bool diagonal, bool pool_materialized = true,
                bool pool_balanced = false) {
  if (!use_hot(flags)) {
    if (!use_hot_f64(flags)) return;
    // the same compile-time flags with the reference's fp64 sigmoid
    v.pass_hot = v.pass_hot_f64;
    v.pass_ahead_hot = v.pass_ahead_hot_f64;
    v.pass_pipe_hot = v.pass_pipe_hot_f64;
    v.pool_hot = v.pool_hot_f64;
    v.pool_hot_diag = v.pool_hot_diag_f64;
    v.pool_bal_hot = v.pool_bal_hot_f64;
    v.pool_bal_hot_diag = v.pool_bal_hot_diag_f64;
    v.pass_staged_hot = v.pass_staged_hot_f64;
  }
  // GB_PASS_AHEAD=1: the KIND 2 throughput pass (index chain one source
  // ahead): +1.3% on C2 but -8% / -10% on C3's second and third levels
  // (high-degree, partly L2-resident), so the inline chain is the default
  static const bool ahead = [] {
    const char *e = std::getenv("GB_PASS_AHEAD");
    return e && std::atoi(e) != 0;
  }();
  if (ahead && v.pass_ahead_hot)
    v.pass = v.pass_ahead_hot;
  else if (v.pass_hot)
    v.pass = v.pass_hot;
  if (v.pass_pipe_hot) v.pass_pipe = v.pass_pipe_hot;
  PoolFn p = pool_balanced ? (diagonal ? v.pool_bal_hot_diag : v.pool_bal_hot)
                           : (diagonal ? v.pool_hot_diag : v.pool_hot);
  if (p && (pool_materialized || pool_balanced)) v.pool = p;
}

// Dynamic shared memory of a KIND 0/2 pass or pair-side launch: one slot per
// group for the source's initial copy (SrcKeep) on vector layouts.
size_t s0_bytes(const Variant &var, int dim) {
  return var.s0_smem ? (size_t)(kBlock / var.G) * dim * sizeof(float) : 0;
}

// Launch of a pair-side kernel.
int launch_pool(const Variant &var, const PoolArgs &a, int grid, cudaStream_t st) {
  var.pool<<<grid, kBlock, s0_bytes(var, a.dim), st>>>(a);
  GB_CHECK_LAUNCH();
  return GB_OK;
}

bool aligned16(const void *p, int dim) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0 && dim % 4 == 0;
}

int grid_for(const void *sym, int G, int64_t max_groups, int64_t work_items, int *grid,
             size_t smem = 0) {
  int occ = 0;
  GB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sym, kBlock, smem));
  if (occ < 1) occ = 1;
  const int64_t groups_per_block = kBlock / G;
  const int64_t want = (int64_t)num_sms() * occ;
  int64_t cap_groups = max_groups > 0 ? max_groups : INT64_MAX;
  cap_groups = std::min(cap_groups, std::max<int64_t>(work_items, 1));
  const int64_t need = (cap_groups + groups_per_block - 1) / groups_per_block;
  *grid = (int)std::max<int64_t>(1, std::min(want, need));
  return GB_OK;
}

}  // namespace
}  // namespace tk
}  // namespace gb

using namespace gb;
using namespace gb::tk;

static int train_passes_impl(int64_t num_vertices, const int64_t *xadj, const int32_t *adj,
                             const int32_t *sources, int64_t n_sources, float *M, int dim,
                             int n_neg, uint64_t seed, uint64_t rng_stream, int64_t pass_begin,
                             int64_t n_passes, int64_t passes_per_epoch,
                             const float *lr_per_epoch, unsigned flags, int64_t max_groups,
                             int64_t *status, double ppr_alpha, void *stream_handle) {
  GB_REQUIRE(num_vertices >= 0 && dim >= 1 && n_neg >= 0, "gb_train_passes: bad sizes");
  GB_REQUIRE(ppr_alpha >= 0.0 && ppr_alpha < 1.0, "gb_train_passes: ppr_alpha in [0, 1)");
  // PPR positives run on the run-time-flag kernels (the HOT ones draw
  // adjacency positives only)
  const bool ppr = ppr_alpha > 0.0;
  GB_REQUIRE(passes_per_epoch >= 1 && pass_begin >= 0 && n_passes >= 0,
             "gb_train_passes: bad pass range");
  GB_REQUIRE(xadj && M && lr_per_epoch && status, "gb_train_passes: null pointer");
  if (num_vertices == 0 || n_passes == 0) return GB_OK;
  const bool exact = flags & GB_TRAIN_EXACT;
  Variant var;
  GB_REQUIRE(pick_variant(dim, aligned16(M, dim), exact, var),
             "gb_train_passes: dim %d unsupported", dim);
  if (!ppr) select_hot(var, flags, false);
  GB_REQUIRE(!sources || n_sources >= 0, "gb_train_passes: bad source list");
  PassArgs a{num_vertices, xadj, adj, sources, n_sources, M, dim, n_neg, seed, rng_stream, pass_begin, n_passes,
             passes_per_epoch, lr_per_epoch, (flags & GB_TRAIN_REUSE) != 0,
             (flags & GB_TRAIN_FAST_SIGMOID) != 0, !exact && (flags & GB_TRAIN_ATOMIC) != 0,
             (float)ppr_alpha, exact ? 1 : max_groups, status};
  int grid = 1, block = kBlock;
  size_t smem = s0_bytes(var, dim);
  PassFn fn = var.pass;
  if (!exact) {
    const int64_t items = sources ? n_sources : num_vertices;
    int rc = grid_for((const void *)var.pass, var.G, max_groups, items, &grid, smem);
    if (rc) return rc;
    // Uncapped launches (the cap reaches the throughput variant's full
    // occupancy) run KIND 3: sample rows staged in shared memory by cp.async,
    // 80 registers, 3 blocks per SM -- C2 5.34 vs 5.13 G upd/s, C3's
    // uncapped levels unchanged; capped mid-size levels lose (3.35 vs 4.28 at
    // C3 L2: per-source latency, not occupancy, bounds them), so they keep
    // KIND 0.  GB_PASS_SMEM=0 disables, =1 forces.
    {
      int occ0 = 0;
      GB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ0, (const void *)var.pass,
                                                                kBlock, smem));
      const int64_t full0 = (int64_t)num_sms() * std::max(occ0, 1) * (kBlock / var.G);
      const int64_t want = std::min<int64_t>(max_groups > 0 ? max_groups : INT64_MAX, items);
      const char *env = std::getenv("GB_PASS_SMEM");
      const bool on = env ? std::atoi(env) != 0 : want >= full0;
      // (select_hot swapped in the fp64-sigmoid instantiations without
      // GB_TRAIN_FAST_SIGMOID)
      if (on && var.pass_staged_hot && (use_hot(flags) || use_hot_f64(flags)) && !ppr)
        var.pass = var.pass_staged_hot;
      else if (on && ppr && var.pass_staged_hot_ppr && use_hot_f64(flags))
        var.pass = var.pass_staged_hot_ppr;  // PPR walk in the staged HOT pass
      fn = var.pass;
    }
    const bool staged = var.pass && (var.pass == var.pass_staged_hot ||
                                     var.pass == var.pass_staged_hot_ppr);
    if (staged) {
      smem = (size_t)(kBlock / var.G) * kChunk * dim * sizeof(float);
      GB_CUDA_TRY(cudaFuncSetAttribute((const void *)var.pass,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int occ_s = 0;
      GB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, (const void *)var.pass,
                                                                kBlock, smem));
      const int64_t gpb = kBlock / var.G;
      int64_t cap = max_groups > 0 ? max_groups : INT64_MAX;
      cap = std::min(cap, std::max<int64_t>(items, 1));
      grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms() * std::max(occ_s, 1),
                                                         (cap + gpb - 1) / gpb));
    }
    // A launch whose in-flight cap is below what the throughput variant holds
    // on the GPU is latency-bound (small levels): switch to the latency
    // variant -- widest lane layout, batched index fetch and batched dots,
    // one warp per block so the groups spread over all SMs -- when the cap
    // fits its capacity.  GB_PIPE=0/1 forces the choice for experiments.
    int occ = 0;
    GB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)var.pass,
                                                              kBlock, smem));
    const int64_t full = (int64_t)num_sms() * std::max(occ, 1) * (kBlock / var.G);
    const int64_t groups = std::min<int64_t>(max_groups > 0 ? max_groups : INT64_MAX, items);
    Variant lat;
    bool pipe = false;
    int occ1 = 0;
    if (groups < full && pick_variant(dim, aligned16(M, dim), exact, lat, true)) {
      if (!ppr) select_hot(lat, flags, false);
      GB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &occ1, (const void *)lat.pass_pipe, 32, 0));
      pipe = groups <= (int64_t)num_sms() * std::max(occ1, 1) * (32 / lat.G);
    }
    if (const char *env = std::getenv("GB_PIPE")) {
      pipe = std::atoi(env) != 0 && pick_variant(dim, aligned16(M, dim), exact, lat, true);
      if (pipe && !ppr) select_hot(lat, flags, false);
      if (pipe)
        GB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &occ1, (const void *)lat.pass_pipe, 32, 0));
    }
    if (pipe) {
      fn = lat.pass_pipe;
      const int64_t gpw = 32 / lat.G;
      const int64_t warps = std::max<int64_t>(1, (groups + gpw - 1) / gpw);
      grid = (int)std::min<int64_t>(warps, (int64_t)num_sms() * std::max(occ1, 1));
      block = 32;
      smem = 0;
    }
  } else {
    block = 32;
  }
  fn<<<grid, block, smem, as_stream(stream_handle)>>>(a);
  GB_CHECK_LAUNCH();
  return GB_OK;
}

GB_API int gb_train_passes(int64_t num_vertices, const int64_t *xadj, const int32_t *adj,
                           const int32_t *sources, int64_t n_sources, float *M, int dim,
                           int n_neg, uint64_t seed, uint64_t rng_stream, int64_t pass_begin,
                           int64_t n_passes, int64_t passes_per_epoch,
                           const float *lr_per_epoch, unsigned flags, int64_t max_groups,
                           int64_t *status, void *stream_handle) {
  return train_passes_impl(num_vertices, xadj, adj, sources, n_sources, M, dim, n_neg, seed,
                           rng_stream, pass_begin, n_passes, passes_per_epoch, lr_per_epoch,
                           flags, max_groups, status, 0.0, stream_handle);
}

GB_API int gb_train_passes_ppr(int64_t num_vertices, const int64_t *xadj, const int32_t *adj,
                               const int32_t *sources, int64_t n_sources, float *M, int dim,
                               int n_neg, uint64_t seed, uint64_t rng_stream,
                               int64_t pass_begin, int64_t n_passes, int64_t passes_per_epoch,
                               const float *lr_per_epoch, unsigned flags, int64_t max_groups,
                               int64_t *status, double ppr_alpha, void *stream_handle) {
  GB_REQUIRE(ppr_alpha > 0.0, "gb_train_passes_ppr: ppr_alpha must be > 0");
  return train_passes_impl(num_vertices, xadj, adj, sources, n_sources, M, dim, n_neg, seed,
                           rng_stream, pass_begin, n_passes, passes_per_epoch, lr_per_epoch,
                           flags, max_groups, status, ppr_alpha, stream_handle);
}

static int train_pool_side_impl(float *Msrc, float *Mtgt, int dim, const int32_t *targets,
                                int64_t n_src, int B, int64_t lo_t, int64_t n_t, int n_neg,
                                double lr, uint64_t seed, uint64_t side, const int64_t *xadj,
                                const int32_t *adj, int64_t lo_s, uint64_t pool_side,
                                unsigned flags, int64_t max_groups, int64_t *status,
                                const PairParam *param, void *stream_handle) {
  GB_REQUIRE(dim >= 1 && B >= 1 && n_neg >= 0 && n_src >= 0 && n_t >= 0,
             "gb_train_pool_side: bad sizes");
  GB_REQUIRE(Msrc && Mtgt && status, "gb_train_pool_side: null pointer");
  GB_REQUIRE(targets || (xadj && adj), "gb_train_pool_side: need targets or a CSR");
  if (n_src == 0 || n_t == 0) return GB_OK;
  const bool exact = flags & GB_TRAIN_EXACT;
  Variant var;
  GB_REQUIRE(pick_variant(dim, aligned16(Msrc, dim) && aligned16(Mtgt, dim), exact, var),
             "gb_train_pool_side: dim %d unsupported", dim);
  select_hot(var, flags, Msrc == Mtgt, targets != nullptr);
  PoolArgs a{Msrc, Mtgt, dim, targets, n_src, B, lo_t, n_t, n_neg, lr, seed, side, xadj, adj,
             lo_s, pool_side, nullptr, nullptr, nullptr, nullptr, nullptr, (flags & GB_TRAIN_REUSE) != 0,
             (flags & GB_TRAIN_FAST_SIGMOID) != 0, !exact && (flags & GB_TRAIN_ATOMIC) != 0, exact ? 1 : max_groups, status, param};
  int grid = 1;
  if (!exact) {
    int rc = grid_for((const void *)var.pool, var.G, max_groups, n_src, &grid, s0_bytes(var, dim));
    if (rc) return rc;
  }
  return launch_pool(var, a, grid, as_stream(stream_handle));
}

GB_API int gb_train_pool_side(float *Msrc, float *Mtgt, int dim, const int32_t *targets,
                              int64_t n_src, int B, int64_t lo_t, int64_t n_t, int n_neg,
                              double lr, uint64_t seed, uint64_t side, const int64_t *xadj,
                              const int32_t *adj, int64_t lo_s, uint64_t pool_side,
                              unsigned flags, int64_t max_groups, int64_t *status,
                              void *stream_handle) {
  return train_pool_side_impl(Msrc, Mtgt, dim, targets, n_src, B, lo_t, n_t, n_neg, lr, seed,
                              side, xadj, adj, lo_s, pool_side, flags, max_groups, status,
                              nullptr, stream_handle);
}

GB_API int gb_train_pool_side_dp(float *Msrc, float *Mtgt, int dim, const int32_t *targets,
                                 int64_t n_src, int B, int64_t lo_t, int64_t n_t, int n_neg,
                                 const void *param, uint64_t side, const int64_t *xadj,
                                 const int32_t *adj, int64_t lo_s, uint64_t pool_side,
                                 unsigned flags, int64_t max_groups, int64_t *status,
                                 void *stream_handle) {
  GB_REQUIRE(param, "gb_train_pool_side_dp: null param");
  return train_pool_side_impl(Msrc, Mtgt, dim, targets, n_src, B, lo_t, n_t, n_neg, 0.0, 0,
                              side, xadj, adj, lo_s, pool_side, flags, max_groups, status,
                              static_cast<const PairParam *>(param), stream_handle);
}

static int train_pool_list_impl(float *Msrc, float *Mtgt, int dim, const int32_t *list,
                                const int32_t *targets, const int64_t *count, int64_t max_src,
                                int B, int64_t lo_t, int64_t n_t, int n_neg, double lr,
                                uint64_t seed, uint64_t side, unsigned flags, int64_t max_groups,
                                int64_t *status, const PairParam *param, void *stream_handle) {
  GB_REQUIRE(dim >= 1 && B >= 1 && n_neg >= 0 && max_src >= 0 && n_t >= 0,
             "gb_train_pool_list: bad sizes");
  GB_REQUIRE(Msrc && Mtgt && status && list && targets && count,
             "gb_train_pool_list: null pointer");
  if (max_src == 0 || n_t == 0) return GB_OK;
  const bool exact = flags & GB_TRAIN_EXACT;
  Variant var;
  GB_REQUIRE(pick_variant(dim, aligned16(Msrc, dim) && aligned16(Mtgt, dim), exact, var),
             "gb_train_pool_list: dim %d unsupported", dim);
  select_hot(var, flags, Msrc == Mtgt);
  PoolArgs a{Msrc, Mtgt, dim, targets, max_src, B, lo_t, n_t, n_neg, lr, seed, side, nullptr,
             nullptr, 0, 0, list, count, nullptr, nullptr, nullptr, (flags & GB_TRAIN_REUSE) != 0,
             (flags & GB_TRAIN_FAST_SIGMOID) != 0, !exact && (flags & GB_TRAIN_ATOMIC) != 0,
             exact ? 1 : max_groups, status, param};
  int grid = 1;
  if (!exact) {
    int rc = grid_for((const void *)var.pool, var.G, max_groups, max_src, &grid, s0_bytes(var, dim));
    if (rc) return rc;
  }
  return launch_pool(var, a, grid, as_stream(stream_handle));
}

static int train_pool_balanced_impl(float *Msrc, float *Mtgt, int dim, const int32_t *list,
                                    const int64_t *first, const int32_t *cnt, const int32_t *npos,
                                    const int64_t *count, int64_t max_src, int B, int64_t lo_t,
                                    int64_t n_t, int n_neg, double lr, uint64_t seed,
                                    uint64_t side, const int32_t *adj, int64_t lo_s,
                                    uint64_t pool_side, unsigned flags, int64_t max_groups,
                                    int64_t *status, const PairParam *param,
                                    void *stream_handle) {
  GB_REQUIRE(dim >= 1 && B >= 1 && n_neg >= 0 && max_src >= 0 && n_t >= 0,
             "gb_train_pool_balanced: bad sizes");
  GB_REQUIRE(Msrc && Mtgt && status && list && first && cnt && npos && count && adj,
             "gb_train_pool_balanced: null pointer");
  if (max_src == 0 || n_t == 0) return GB_OK;
  const bool exact = flags & GB_TRAIN_EXACT;
  Variant var;
  GB_REQUIRE(pick_variant(dim, aligned16(Msrc, dim) && aligned16(Mtgt, dim), exact, var),
             "gb_train_pool_balanced: dim %d unsupported", dim);
  select_hot(var, flags, Msrc == Mtgt, false, true);
  PoolArgs a{Msrc, Mtgt, dim, nullptr, max_src, B, lo_t, n_t, n_neg, lr, seed, side, nullptr,
             adj, lo_s, pool_side, list, count, first, cnt, npos,
             (flags & GB_TRAIN_REUSE) != 0, (flags & GB_TRAIN_FAST_SIGMOID) != 0,
             !exact && (flags & GB_TRAIN_ATOMIC) != 0, exact ? 1 : max_groups, status, param};
  int grid = 1;
  if (!exact) {
    int rc = grid_for((const void *)var.pool, var.G, max_groups, max_src, &grid, s0_bytes(var, dim));
    if (rc) return rc;
  }
  return launch_pool(var, a, grid, as_stream(stream_handle));
}

GB_API int gb_train_pool_list(float *Msrc, float *Mtgt, int dim, const int32_t *list,
                              const int32_t *targets, const int64_t *count, int64_t max_src,
                              int B, int64_t lo_t, int64_t n_t, int n_neg, double lr,
                              uint64_t seed, uint64_t side, unsigned flags, int64_t max_groups,
                              int64_t *status, void *stream_handle) {
  return train_pool_list_impl(Msrc, Mtgt, dim, list, targets, count, max_src, B, lo_t, n_t,
                              n_neg, lr, seed, side, flags, max_groups, status, nullptr,
                              stream_handle);
}

GB_API int gb_train_pool_list_dp(float *Msrc, float *Mtgt, int dim, const int32_t *list,
                                 const int32_t *targets, const int64_t *count, int64_t max_src,
                                 int B, int64_t lo_t, int64_t n_t, int n_neg, const void *param,
                                 uint64_t side, unsigned flags, int64_t max_groups,
                                 int64_t *status, void *stream_handle) {
  GB_REQUIRE(param, "gb_train_pool_list_dp: null param");
  return train_pool_list_impl(Msrc, Mtgt, dim, list, targets, count, max_src, B, lo_t, n_t,
                              n_neg, 0.0, 0, side, flags, max_groups, status,
                              static_cast<const PairParam *>(param), stream_handle);
}

GB_API int gb_train_pool_balanced(float *Msrc, float *Mtgt, int dim, const int32_t *list,
                                  const int64_t *first, const int32_t *cnt, const int32_t *npos,
                                  const int64_t *count, int64_t max_src, int B, int64_t lo_t,
                                  int64_t n_t, int n_neg, double lr, uint64_t seed,
                                  uint64_t side, const int32_t *adj, int64_t lo_s,
                                  uint64_t pool_side, unsigned flags, int64_t max_groups,
                                  int64_t *status, void *stream_handle) {
  return train_pool_balanced_impl(Msrc, Mtgt, dim, list, first, cnt, npos, count, max_src, B,
                                  lo_t, n_t, n_neg, lr, seed, side, adj, lo_s, pool_side, flags,
                                  max_groups, status, nullptr, stream_handle);
}

GB_API int gb_train_pool_balanced_dp(float *Msrc, float *Mtgt, int dim, const int32_t *list,
                                     const int64_t *first, const int32_t *cnt,
                                     const int32_t *npos, const int64_t *count, int64_t max_src,
                                     int B, int64_t lo_t, int64_t n_t, int n_neg,
                                     const void *param, uint64_t side, const int32_t *adj,
                                     int64_t lo_s, uint64_t pool_side, unsigned flags,
                                     int64_t max_groups, int64_t *status, void *stream_handle) {
  GB_REQUIRE(param, "gb_train_pool_balanced_dp: null param");
  return train_pool_balanced_impl(Msrc, Mtgt, dim, list, first, cnt, npos, count, max_src, B,
                                  lo_t, n_t, n_neg, 0.0, 0, side, adj, lo_s, pool_side, flags,
                                  max_groups, status, static_cast<const PairParam *>(param),
                                  stream_handle);
}

GB_API int gb_nonfinite_scan(const float *M, int64_t count, int64_t epoch, int64_t *status,
                                 void *stream_handle) {
  GB_REQUIRE(count >= 0 && status, "gb_nonfinite_scan: bad args");
  if (count == 0) return GB_OK;
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, (int64_t)num_sms() * 8);
  nonfinite_scan_kernel<<<(int)blocks, 256, 0, as_stream(stream_handle)>>>(M, count, epoch,
                                                                           status);
  GB_CHECK_LAUNCH();
  return GB_OK;
}

GB_API int gb_apply_sample_lists(float *M, int dim, int64_t n_src, const int64_t *src, int k,
                                 const int64_t *samples, const int8_t *labels, double lr,
                                 unsigned flags, int64_t max_groups, int64_t *status,
                                 void *stream_handle) {
  GB_REQUIRE(M && dim >= 1 && n_src >= 0 && k >= 0 && status, "gb_apply_sample_lists: bad args");
  GB_REQUIRE(n_src == 0 || (src && (k == 0 || (samples && labels))),
             "gb_apply_sample_lists: null pointer");
  if (n_src == 0) return GB_OK;
  const bool exact = flags & GB_TRAIN_EXACT;
  Variant var;
  GB_REQUIRE(pick_variant(dim, aligned16(M, dim), exact, var),
             "gb_apply_sample_lists: dim %d unsupported", dim);
  ListArgs a{M, dim, n_src, src, k, samples, labels, lr, (flags & GB_TRAIN_REUSE) != 0,
             (flags & GB_TRAIN_FAST_SIGMOID) != 0, !exact && (flags & GB_TRAIN_ATOMIC) != 0, exact ? 1 : max_groups, status};
  int grid = 1;
  if (!exact) {
    int rc = grid_for((const void *)var.lists, var.G, max_groups, n_src, &grid);
    if (rc) return rc;
  }
  var.lists<<<grid, kBlock, 0, as_stream(stream_handle)>>>(a);
  GB_CHECK_LAUNCH();
  return GB_OK;
}

namespace gb {
namespace tk {
namespace {
// _fill_pool_side (bigtrain.py:164-196): one thread per source vertex.
__global__ void fill_pool_kernel(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                                 int64_t lo_s, int64_t hi_s, int64_t lo_t, int64_t hi_t, int B,
                                 uint64_t seed, uint64_t side, int32_t *__restrict__ out,
                                 const PairParam *__restrict__ param) {
  if (param) seed = param->seed;
  for (int64_t v = lo_s + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < hi_s;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e1 = xadj[v + 1];
    const int64_t first = lower_bound_adj(adj, xadj[v], e1, lo_t);
    const int64_t cnt = lower_bound_adj(adj, first, e1, hi_t) - first;
    const uint64_t key = stream_key(seed, side, 0, (uint64_t)v);
    int32_t *row = out + (v - lo_s) * B;
    for (int t = 0; t < B; ++t)
      row[t] = cnt > 0 ? adj[first + draw_below(key, (uint64_t)t, cnt)] : -1;
  }
}

// Compacted pool side: the same draws as fill_pool_kernel, but only sources
// with a neighbour in [lo_t, hi_t) get an entry (list[k] = v - lo_s, pool
// row targets[k*B ..]); warp-aggregated append, so entries of one warp stay
// in id order while warps land in any order (Hogwild launches do not depend
// on source order).  Sources without such a neighbour train nothing
// (bigtrain.py:229-231), so the pair kernel never sees them.
__global__ void fill_pool_compact_kernel(const int64_t *__restrict__ xadj,
                                         const int32_t *__restrict__ adj, int64_t lo_s,
                                         int64_t hi_s, int64_t lo_t, int64_t hi_t, int B,
                                         uint64_t seed, uint64_t side, int32_t *__restrict__ list,
                                         int32_t *__restrict__ targets,
                                         unsigned long long *count,
                                         const PairParam *__restrict__ param) {
  const int lane = threadIdx.x & 31;
  if (param) seed = param->seed;
  for (int64_t v0 = lo_s + (int64_t)blockIdx.x * blockDim.x; v0 < hi_s;
       v0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = v0 + threadIdx.x;
    int64_t first = 0, cnt = 0;
    if (v < hi_s) {
      const int64_t e1 = __ldg(xadj + v + 1);
      first = lower_bound_adj(adj, __ldg(xadj + v), e1, lo_t);
      cnt = lower_bound_adj(adj, first, e1, hi_t) - first;
    }
    const unsigned m = __ballot_sync(0xffffffffu, cnt > 0);
    if (m == 0) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(count, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (cnt > 0) {
      const int64_t slot = (int64_t)base + __popc(m & ((1u << lane) - 1u));
      list[slot] = (int32_t)(v - lo_s);
      const uint64_t key = stream_key(seed, side, 0, (uint64_t)v);
      int32_t *row = targets + slot * B;
      for (int t = 0; t < B; ++t) row[t] = __ldg(adj + first + draw_below(key, (uint64_t)t, cnt));
    }
  }
}

// Balanced pool side: every source with a neighbour anywhere gets an entry;
// its positives in this pair number npos = floor(BK*cnt/deg + u), u uniform
// from key(seed, side, 2, v) -- in expectation the share of BK positives
// (B per pass-equivalent, K parts) that the in-memory pass would draw from
// the part's cnt of its deg neighbours.  Positives are drawn in the pair
// kernel from adj[first .. first + cnt).
__global__ void fill_pool_balanced_kernel(const int64_t *__restrict__ xadj,
                                          const int32_t *__restrict__ adj, int64_t lo_s,
                                          int64_t hi_s, int64_t lo_t, int64_t hi_t, int64_t BK,
                                          uint64_t seed, uint64_t side,
                                          int32_t *__restrict__ list, int64_t *__restrict__ first,
                                          int32_t *__restrict__ cnt_out,
                                          int32_t *__restrict__ npos_out,
                                          unsigned long long *count,
                                          const PairParam *__restrict__ param) {
  const int lane = threadIdx.x & 31;
  if (param) seed = param->seed;
  for (int64_t v0 = lo_s + (int64_t)blockIdx.x * blockDim.x; v0 < hi_s;
       v0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = v0 + threadIdx.x;
    int64_t f = 0, cnt = 0, deg = 0;
    if (v < hi_s) {
      const int64_t e0 = __ldg(xadj + v), e1 = __ldg(xadj + v + 1);
      deg = e1 - e0;
      if (deg > 0) {
        f = lower_bound_adj(adj, e0, e1, lo_t);
        cnt = lower_bound_adj(adj, f, e1, hi_t) - f;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, deg > 0);
    if (m == 0) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(count, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (deg > 0) {
      const int64_t slot = (int64_t)base + __popc(m & ((1u << lane) - 1u));
      const double share = __ddiv_rn((double)(BK * cnt), (double)deg);
      const double u = draw_unit(stream_key(seed, side, 2, (uint64_t)v), 0);
      list[slot] = (int32_t)(v - lo_s);
      first[slot] = f;
      cnt_out[slot] = (int32_t)cnt;
      npos_out[slot] = cnt > 0 ? (int32_t)floor(__dadd_rn(share, u)) : 0;
    }
  }
}
}  // namespace
}  // namespace tk
}  // namespace gb

static int fill_pool_balanced_impl(const int64_t *xadj, const int32_t *adj, int64_t lo_s,
                                   int64_t hi_s, int64_t lo_t, int64_t hi_t, int64_t BK,
                                   uint64_t seed, uint64_t side, int32_t *list, int64_t *first,
                                   int32_t *cnt, int32_t *npos, int64_t *count,
                                   const PairParam *param, void *stream_handle) {
  GB_REQUIRE(xadj && adj && list && first && cnt && npos && count && BK >= 1 &&
                 hi_s >= lo_s && hi_t >= lo_t,
             "gb_fill_pool_balanced: bad args");
  GB_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int64_t), as_stream(stream_handle)));
  const int64_t n = hi_s - lo_s;
  if (n == 0) return GB_OK;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  gb::tk::fill_pool_balanced_kernel<<<(int)blocks, 256, 0, as_stream(stream_handle)>>>(
      xadj, adj, lo_s, hi_s, lo_t, hi_t, BK, seed, side, list, first, cnt, npos,
      reinterpret_cast<unsigned long long *>(count), param);
  GB_CHECK_LAUNCH();
  return GB_OK;
}

static int fill_pool_compact_impl(const int64_t *xadj, const int32_t *adj, int64_t lo_s,
                                  int64_t hi_s, int64_t lo_t, int64_t hi_t, int B, uint64_t seed,
                                  uint64_t side, int32_t *list, int32_t *targets, int64_t *count,
                                  const PairParam *param, void *stream_handle) {
  GB_REQUIRE(xadj && adj && list && targets && count && B >= 1 && hi_s >= lo_s && hi_t >= lo_t,
             "gb_fill_pool_compact: bad args");
  GB_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int64_t), as_stream(stream_handle)));
  const int64_t n = hi_s - lo_s;
  if (n == 0) return GB_OK;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  gb::tk::fill_pool_compact_kernel<<<(int)blocks, 256, 0, as_stream(stream_handle)>>>(
      xadj, adj, lo_s, hi_s, lo_t, hi_t, B, seed, side, list, targets,
      reinterpret_cast<unsigned long long *>(count), param);
  GB_CHECK_LAUNCH();
  return GB_OK;
}

GB_API int gb_fill_pool_balanced(const int64_t *xadj, const int32_t *adj, int64_t lo_s,
                                 int64_t hi_s, int64_t lo_t, int64_t hi_t, int64_t BK,
                                 uint64_t seed, uint64_t side, int32_t *list, int64_t *first,
                                 int32_t *cnt, int32_t *npos, int64_t *count,
                                 void *stream_handle) {
  return fill_pool_balanced_impl(xadj, adj, lo_s, hi_s, lo_t, hi_t, BK, seed, side, list, first,
                                 cnt, npos, count, nullptr, stream_handle);
}

GB_API int gb_fill_pool_balanced_dp(const int64_t *xadj, const int32_t *adj, int64_t lo_s,
                                    int64_t hi_s, int64_t lo_t, int64_t hi_t, int64_t BK,
                                    const void *param, uint64_t side, int32_t *list,
                                    int64_t *first, int32_t *cnt, int32_t *npos, int64_t *count,
                                    void *stream_handle) {
  GB_REQUIRE(param, "gb_fill_pool_balanced_dp: null param");
  return fill_pool_balanced_impl(xadj, adj, lo_s, hi_s, lo_t, hi_t, BK, 0, side, list, first,
                                 cnt, npos, count, static_cast<const PairParam *>(param),
                                 stream_handle);
}

GB_API int gb_fill_pool_compact(const int64_t *xadj, const int32_t *adj, int64_t lo_s,
                                int64_t hi_s, int64_t lo_t, int64_t hi_t, int B, uint64_t seed,
                                uint64_t side, int32_t *list, int32_t *targets, int64_t *count,
                                void *stream_handle) {
  return fill_pool_compact_impl(xadj, adj, lo_s, hi_s, lo_t, hi_t, B, seed, side, list, targets,
                                count, nullptr, stream_handle);
}

GB_API int gb_fill_pool_compact_dp(const int64_t *xadj, const int32_t *adj, int64_t lo_s,
                                   int64_t hi_s, int64_t lo_t, int64_t hi_t, int B,
                                   const void *param, uint64_t side, int32_t *list,
                                   int32_t *targets, int64_t *count, void *stream_handle) {
  GB_REQUIRE(param, "gb_fill_pool_compact_dp: null param");
  return fill_pool_compact_impl(xadj, adj, lo_s, hi_s, lo_t, hi_t, B, 0, side, list, targets,
                                count, static_cast<const PairParam *>(param), stream_handle);
}

static int fill_pool_side_impl(const int64_t *xadj, const int32_t *adj, int64_t lo_s,
                               int64_t hi_s, int64_t lo_t, int64_t hi_t, int B, uint64_t seed,
                               uint64_t side, int32_t *out, const PairParam *param,
                               void *stream_handle) {
  GB_REQUIRE(xadj && out && B >= 1 && hi_s >= lo_s && hi_t >= lo_t,
             "gb_fill_pool_side: bad args");
  const int64_t n = hi_s - lo_s;
  if (n == 0) return GB_OK;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  gb::tk::fill_pool_kernel<<<(int)blocks, 256, 0, as_stream(stream_handle)>>>(
      xadj, adj, lo_s, hi_s, lo_t, hi_t, B, seed, side, out, param);
  GB_CHECK_LAUNCH();
  return GB_OK;
}

GB_API int gb_fill_pool_side(const int64_t *xadj, const int32_t *adj, int64_t lo_s, int64_t hi_s,
                             int64_t lo_t, int64_t hi_t, int B, uint64_t seed, uint64_t side,
                             int32_t *out, void *stream_handle) {
  return fill_pool_side_impl(xadj, adj, lo_s, hi_s, lo_t, hi_t, B, seed, side, out, nullptr,
                             stream_handle);
}

GB_API int gb_fill_pool_side_dp(const int64_t *xadj, const int32_t *adj, int64_t lo_s,
                                int64_t hi_s, int64_t lo_t, int64_t hi_t, int B,
                                const void *param, uint64_t side, int32_t *out,
                                void *stream_handle) {
  GB_REQUIRE(param, "gb_fill_pool_side_dp: null param");
  return fill_pool_side_impl(xadj, adj, lo_s, hi_s, lo_t, hi_t, B, 0, side, out,
                             static_cast<const PairParam *>(param), stream_handle);
}
