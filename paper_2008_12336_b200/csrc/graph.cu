// Graph-side kernels: CSR construction (graph.py:93-131), id densification
// (graph.py:160-164), the R-MAT input generator, degree order
// (coarsen.py:69-95), the order-priority MultiEdgeCollapse (coarsen.py:98-114,
// restated in SURVEY.md Appendix B), coarse CSR (coarsen.py:182-281) and the
// coarse-to-fine projection (trainer.py:243-249).
//
// All of it is integer/byte work bounded by HBM: arcs are mapped to 64-bit
// (row, col) keys, radix-sorted, run-length deduplicated and turned into
// row offsets by a per-row binary search -- the sorted unique key sequence IS
// the CSR, so the result is bit-identical to the reference's numpy/numba
// construction by definition.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace gb {
namespace {

constexpr uint64_t kRmatStream = 0x524D4154ull;  // "RMAT"
constexpr uint64_t kPermStream = 0x5045524Dull;  // "PERM"
constexpr int8_t kUndecided = 0, kHub = 1, kMember = 2;

// Carves 256-byte aligned sub-buffers out of a caller workspace.  With a
// null base it only accumulates the size (workspace queries).
struct Carver {
  char *base;
  size_t off = 0;
  explicit Carver(void *b) : base(static_cast<char *>(b)) {}
  template <class T>
  T *take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
  void *take_bytes(size_t n) { return take<char>(n); }
};

inline int bits_for(uint64_t x) {  // number of bits to represent values <= x
  int b = 0;
  while (b < 64 && (x >> b) != 0) ++b;
  return std::max(b, 1);
}

inline int blocks_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 32;
  return (int)std::max<int64_t>(1, std::min(b, cap));
}

#define GRID_STRIDE(i, n)                                                   \
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); \
       i += (int64_t)gridDim.x * blockDim.x)

// ---------------------------------------------------------------------------
// sorted-key -> CSR helpers
// ---------------------------------------------------------------------------
__global__ void keys_from_arcs(const int64_t *__restrict__ src, const int64_t *__restrict__ dst,
                               int64_t n, int64_t V, bool drop_self, bool sym, uint64_t sentinel,
                               uint64_t *__restrict__ keys) {
  GRID_STRIDE(i, n) {
    const int64_t s = src[i], d = dst[i];
    const bool self = drop_self && s == d;
    keys[i] = self ? sentinel : (uint64_t)s * (uint64_t)V + (uint64_t)d;
    if (sym) keys[n + i] = self ? sentinel : (uint64_t)d * (uint64_t)V + (uint64_t)s;
  }
}

// xadj[r] = lower_bound(keys, r*V) over the sorted unique keys.
__global__ void xadj_from_keys(const uint64_t *__restrict__ keys, int64_t nkeys, int64_t V,
                               int64_t *__restrict__ xadj) {
  GRID_STRIDE(r, V + 1) {
    const uint64_t target = (uint64_t)r * (uint64_t)V;
    int64_t lo = 0, hi = nkeys;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target)
        lo = mid + 1;
      else
        hi = mid;
    }
    xadj[r] = lo;
  }
}

__global__ void adj_from_keys(const uint64_t *__restrict__ keys, int64_t nkeys, int64_t V,
                              int32_t *__restrict__ adj) {
  GRID_STRIDE(i, nkeys) adj[i] = (int32_t)(keys[i] % (uint64_t)V);
}

// Sort keys, deduplicate, strip the sentinel tail, emit xadj/adj.  Shared by
// the CSR build and the coarse-graph build.
struct KeyCsrBuffers {
  uint64_t *keys_alt;
  uint64_t *uniq;
  int64_t *num_sel;
  void *cub_tmp;
  size_t cub_bytes;
};

int key_csr_carve(Carver &c, int64_t n, int end_bit, KeyCsrBuffers &b) {
  b.keys_alt = c.take<uint64_t>(n);
  b.uniq = c.take<uint64_t>(n);
  b.num_sel = c.take<int64_t>(1);
  size_t sort_bytes = 0, uniq_bytes = 0;
  GB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, (uint64_t *)nullptr,
                                             (uint64_t *)nullptr, n, 0, end_bit));
  GB_CUDA_TRY(cub::DeviceSelect::Unique(nullptr, uniq_bytes, (uint64_t *)nullptr,
                                        (uint64_t *)nullptr, (int64_t *)nullptr, n));
  b.cub_bytes = std::max(sort_bytes, uniq_bytes);
  b.cub_tmp = c.take_bytes(b.cub_bytes);
  return GB_OK;
}

int keys_to_csr(uint64_t *keys, int64_t n, int end_bit, int64_t V, uint64_t sentinel,
                KeyCsrBuffers &b, int64_t *xadj, int32_t *adj, int64_t *num_edges_out,
                cudaStream_t st) {
  int64_t nuniq = 0;
  if (n > 0) {
    size_t tb = b.cub_bytes;
    GB_CUDA_TRY(
        cub::DeviceRadixSort::SortKeys(b.cub_tmp, tb, keys, b.keys_alt, n, 0, end_bit, st));
    tb = b.cub_bytes;
    GB_CUDA_TRY(cub::DeviceSelect::Unique(b.cub_tmp, tb, b.keys_alt, b.uniq, b.num_sel, n, st));
    GB_CUDA_TRY(cudaMemcpyAsync(&nuniq, b.num_sel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GB_CUDA_TRY(cudaStreamSynchronize(st));
    if (nuniq > 0) {
      uint64_t last = 0;
      GB_CUDA_TRY(cudaMemcpyAsync(&last, b.uniq + nuniq - 1, sizeof(uint64_t),
                                  cudaMemcpyDeviceToHost, st));
      GB_CUDA_TRY(cudaStreamSynchronize(st));
      if (last == sentinel) --nuniq;
    }
  }
  xadj_from_keys<<<blocks_for(V + 1), 256, 0, st>>>(b.uniq, nuniq, V, xadj);
  GB_CHECK_LAUNCH();
  if (nuniq > 0) {
    adj_from_keys<<<blocks_for(nuniq), 256, 0, st>>>(b.uniq, nuniq, V, adj);
    GB_CHECK_LAUNCH();
  }
  GB_CUDA_TRY(cudaStreamSynchronize(st));
  *num_edges_out = nuniq;
  return GB_OK;
}

// ---------------------------------------------------------------------------
// densify
// ---------------------------------------------------------------------------
__global__ void nonisolated_flags(const int64_t *__restrict__ xadj, int64_t V,
                                  int64_t *__restrict__ flag) {
  GRID_STRIDE(v, V) flag[v] = xadj[v + 1] > xadj[v] ? 1 : 0;
}

__global__ void densify_vertices(const int64_t *__restrict__ xadj, const int64_t *__restrict__ pos,
                                 int64_t V, int64_t *__restrict__ new_id,
                                 int64_t *__restrict__ kept, int64_t *__restrict__ xadj_out) {
  GRID_STRIDE(v, V) {
    if (xadj[v + 1] > xadj[v]) {
      const int64_t k = pos[v];
      new_id[v] = k;
      kept[k] = v;
      xadj_out[k] = xadj[v];  // removing empty rows does not move arcs
    } else {
      new_id[v] = -1;
    }
  }
}

__global__ void remap_adj(const int32_t *__restrict__ adj, int64_t E,
                          const int64_t *__restrict__ new_id, int32_t *__restrict__ adj_out) {
  GRID_STRIDE(e, E) adj_out[e] = (int32_t)new_id[adj[e]];
}

__global__ void active_flags(const int64_t *__restrict__ xadj, int64_t V,
                             int32_t *__restrict__ ids, char *__restrict__ flag) {
  GRID_STRIDE(v, V) {
    ids[v] = (int32_t)v;
    flag[v] = xadj[v + 1] > xadj[v];
  }
}

__global__ void set_tail(int64_t *__restrict__ xadj_out, const int64_t *__restrict__ count,
                         int64_t E) {
  xadj_out[*count] = E;
}

// ---------------------------------------------------------------------------
// R-MAT
// ---------------------------------------------------------------------------
__global__ void perm_keys(int64_t n, uint64_t pkey, uint64_t *__restrict__ keys,
                          int64_t *__restrict__ ids) {
  GRID_STRIDE(i, n) {
    keys[i] = draw_u64(pkey, (uint64_t)i);
    ids[i] = i;
  }
}

// samples first .. first + n - 1 (a sample is a pure function of its index)
__global__ void rmat_range_kernel(int scale, int64_t first, int64_t n, double ta, double tab,
                                  double tabc, uint64_t seed, const int64_t *__restrict__ perm,
                                  int64_t *__restrict__ src, int64_t *__restrict__ dst) {
  GRID_STRIDE(i, n) {
    const int64_t e = first + i;
    const uint64_t key = stream_key(seed, kRmatStream, (uint64_t)e, 0);
    int64_t u = 0, v = 0;
    for (int l = 0; l < scale; ++l) {
      const double r = draw_unit(key, (uint64_t)l);
      const int64_t bit = int64_t(1) << (scale - 1 - l);
      if (r < ta) {
      } else if (r < tab) {
        v |= bit;
      } else if (r < tabc) {
        u |= bit;
      } else {
        u |= bit;
        v |= bit;
      }
    }
    src[i] = perm ? perm[u] : u;
    dst[i] = perm ? perm[v] : v;
  }
}

__global__ void rmat_kernel(int scale, int64_t n, double ta, double tab, double tabc,
                            uint64_t seed, const int64_t *__restrict__ perm,
                            int64_t *__restrict__ src, int64_t *__restrict__ dst) {
  GRID_STRIDE(e, n) {
    const uint64_t key = stream_key(seed, kRmatStream, (uint64_t)e, 0);
    int64_t u = 0, v = 0;
    for (int l = 0; l < scale; ++l) {
      const double r = draw_unit(key, (uint64_t)l);
      const int64_t bit = int64_t(1) << (scale - 1 - l);
      if (r < ta) {
      } else if (r < tab) {
        v |= bit;
      } else if (r < tabc) {
        u |= bit;
      } else {
        u |= bit;
        v |= bit;
      }
    }
    src[e] = perm ? perm[u] : u;
    dst[e] = perm ? perm[v] : v;
  }
}

// ---------------------------------------------------------------------------
// degree order
// ---------------------------------------------------------------------------
__global__ void degrees_kernel(const int64_t *__restrict__ xadj, int64_t V,
                               uint64_t *__restrict__ deg, int64_t *__restrict__ ids) {
  GRID_STRIDE(v, V) {
    deg[v] = (uint64_t)(xadj[v + 1] - xadj[v]);
    ids[v] = v;
  }
}

__global__ void invert_degree_keys(uint64_t *__restrict__ deg, int64_t V,
                                   const uint64_t *__restrict__ maxdeg) {
  const uint64_t m = *maxdeg;
  GRID_STRIDE(v, V) deg[v] = m - deg[v];
}

// ---------------------------------------------------------------------------
// collapse: u is a HUB iff no H-in-neighbour is a hub;
// a member joins its minimum-rank hub H-in-neighbour.  H-in-neighbours of u:
// w adjacent to u with rank(w) < rank(u) and (small(w) or small(u)).  A vertex
// that is not small has none (a small w has lower degree, hence higher rank),
// so it is a hub outright.
// ---------------------------------------------------------------------------
__global__ void collapse_init(const int64_t *__restrict__ xadj, const int64_t *__restrict__ order,
                              int64_t V, double delta, int64_t *__restrict__ rank,
                              int8_t *__restrict__ status) {
  GRID_STRIDE(i, V) {
    const int64_t v = order[i];
    rank[v] = i;
    const double deg = (double)(xadj[v + 1] - xadj[v]);
    status[v] = deg <= delta ? kUndecided : kHub;  // coarsen.py:108,111
  }
}

// One Gauss-Seidel round over the undecided vertices.  Reading a neighbour's
// status written in this same round is safe: decisions are monotone.
__global__ void collapse_round(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                               const int64_t *__restrict__ rank, int64_t V,
                               volatile int8_t *status, unsigned long long *undecided) {
  unsigned long long left = 0;
  GRID_STRIDE(u, V) {
    if (status[u] != kUndecided) continue;
    const int64_t ru = rank[u];
    bool any_hub = false, all_member = true;
    for (int64_t e = xadj[u]; e < xadj[u + 1]; ++e) {
      const int64_t w = adj[e];
      if (rank[w] >= ru) continue;
      const int8_t sw = status[w];
      if (sw == kHub) {
        any_hub = true;
        break;
      }
      if (sw != kMember) all_member = false;
    }
    if (any_hub)
      status[u] = kMember;
    else if (all_member)
      status[u] = kHub;
    else
      ++left;
  }
  if (left) atomicAdd(undecided, left);
}

// Exact sequential finish for pathological chains: walk the order once; every
// lower-rank vertex is decided by the time u is reached.  One warp.
__global__ void collapse_tail(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                              const int64_t *__restrict__ rank, const int64_t *__restrict__ order,
                              int64_t V, volatile int8_t *status) {
  const int lane = threadIdx.x;
  for (int64_t i = 0; i < V; ++i) {
    const int64_t u = order[i];
    if (status[u] != kUndecided) continue;
    bool hub_nbr = false;
    for (int64_t e = xadj[u] + lane; e < xadj[u + 1]; e += 32) {
      const int64_t w = adj[e];
      if (rank[w] < i && status[w] == kHub) hub_nbr = true;
    }
    hub_nbr = __any_sync(0xffffffffu, hub_nbr);
    if (lane == 0) status[u] = hub_nbr ? kMember : kHub;
    __syncwarp();
    __threadfence_block();
  }
}

__global__ void hub_flags_by_rank(const int64_t *__restrict__ order,
                                  const int8_t *__restrict__ status, int64_t V,
                                  int64_t *__restrict__ flag) {
  GRID_STRIDE(i, V) flag[i] = status[order[i]] == kHub ? 1 : 0;
}

__global__ void assign_clusters(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                                const int64_t *__restrict__ rank,
                                const int8_t *__restrict__ status,
                                const int64_t *__restrict__ cid_by_rank, int64_t V,
                                int32_t *__restrict__ cmap) {
  GRID_STRIDE(u, V) {
    const int64_t ru = rank[u];
    if (status[u] == kHub) {
      cmap[u] = (int32_t)cid_by_rank[ru];
      continue;
    }
    int64_t best = INT64_MAX;
    for (int64_t e = xadj[u]; e < xadj[u + 1]; ++e) {
      const int64_t w = adj[e];
      const int64_t rw = rank[w];
      if (rw < ru && rw < best && status[w] == kHub) best = rw;
    }
    cmap[u] = (int32_t)cid_by_rank[best];
  }
}

// ---------------------------------------------------------------------------
// coarse CSR keys: warp per vertex, lanes over its arcs (coalesced).
// ---------------------------------------------------------------------------
__global__ void coarse_keys(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                            const int32_t *__restrict__ cmap, int64_t V, uint64_t nc,
                            uint64_t sentinel, uint64_t *__restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < V; v += nwarps) {
    const uint64_t cv = (uint64_t)cmap[v];
    const int64_t e1 = xadj[v + 1];
    for (int64_t e = xadj[v] + lane; e < e1; e += 32) {
      const uint64_t cu = (uint64_t)cmap[adj[e]];
      keys[e] = cu == cv ? sentinel : cv * nc + cu;
    }
  }
}

// ---------------------------------------------------------------------------
// expand
// ---------------------------------------------------------------------------
__global__ void expand_vec4(const float4 *__restrict__ coarse, const int32_t *__restrict__ cmap,
                            int64_t rows, int q, float4 *__restrict__ out) {
  GRID_STRIDE(i, rows * q) {
    const int64_t v = i / q;
    const int64_t c = i - v * q;
    out[i] = __ldg(coarse + (int64_t)cmap[v] * q + c);
  }
}

__global__ void expand_scalar(const float *__restrict__ coarse, const int32_t *__restrict__ cmap,
                              int64_t rows, int dim, float *__restrict__ out) {
  GRID_STRIDE(i, rows * dim) {
    const int64_t v = i / dim;
    const int64_t c = i - v * dim;
    out[i] = __ldg(coarse + (int64_t)cmap[v] * dim + c);
  }
}

__global__ void rng_draw_kernel(uint64_t seed, uint64_t stream, uint64_t step, uint64_t v0,
                                uint64_t ctr, int64_t n, int64_t count, int64_t *out) {
  GRID_STRIDE(i, count) out[i] = draw_below(stream_key(seed, stream, step, v0 + i), ctr, n);
}

}  // namespace
}  // namespace gb

using namespace gb;

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
GB_API int gb_rng_draw_below(uint64_t seed, uint64_t stream, uint64_t step, uint64_t vertex0,
                                 uint64_t counter, int64_t n, int64_t count, int64_t *out,
                                 void *stream_handle) {
  GB_REQUIRE(n > 0 && count >= 0 && out, "gb_rng_draw_below: bad args");
  if (count == 0) return GB_OK;
  rng_draw_kernel<<<blocks_for(count), 256, 0, as_stream(stream_handle)>>>(
      seed, stream, step, vertex0, counter, n, count, out);
  GB_CHECK_LAUNCH();
  return GB_OK;
}

static int csr_build_layout(Carver &c, int64_t V, int64_t num_arcs, unsigned flags,
                            uint64_t **keys, KeyCsrBuffers &b, int *end_bit, uint64_t *sentinel) {
  const int64_t n = num_arcs * ((flags & GB_CSR_SYMMETRIZE) ? 2 : 1);
  *sentinel = (uint64_t)V * (uint64_t)V;
  *end_bit = bits_for(*sentinel);
  *keys = c.take<uint64_t>(n);
  return key_csr_carve(c, n, *end_bit, b);
}

GB_API int gb_csr_build_workspace(int64_t num_vertices, int64_t num_arcs, unsigned flags,
                                      size_t *bytes) {
  GB_REQUIRE(num_vertices >= 1 && num_vertices < (int64_t(1) << 31) && num_arcs >= 0 && bytes,
             "gb_csr_build_workspace: bad args");
  Carver c(nullptr);
  uint64_t *keys;
  KeyCsrBuffers b;
  int end_bit;
  uint64_t sentinel;
  int rc = csr_build_layout(c, num_vertices, num_arcs, flags, &keys, b, &end_bit, &sentinel);
  if (rc) return rc;
  *bytes = c.off + 256;
  return GB_OK;
}

GB_API int gb_csr_build(int64_t num_vertices, const int64_t *src, const int64_t *dst,
                            int64_t num_arcs, unsigned flags, int64_t *xadj, int32_t *adj,
                            int64_t *num_edges_out, void *workspace, size_t ws_bytes,
                            void *stream_handle) {
  GB_REQUIRE(num_vertices >= 1 && num_vertices < (int64_t(1) << 31) && num_arcs >= 0,
             "gb_csr_build: bad sizes");
  GB_REQUIRE(xadj && num_edges_out && (num_arcs == 0 || (src && dst && adj)),
             "gb_csr_build: null pointer");
  Carver c(workspace);
  uint64_t *keys;
  KeyCsrBuffers b;
  int end_bit;
  uint64_t sentinel;
  int rc = csr_build_layout(c, num_vertices, num_arcs, flags, &keys, b, &end_bit, &sentinel);
  if (rc) return rc;
  GB_REQUIRE(c.off <= ws_bytes, "gb_csr_build: workspace %zu < %zu", ws_bytes, c.off);
  cudaStream_t st = as_stream(stream_handle);
  const int64_t n = num_arcs * ((flags & GB_CSR_SYMMETRIZE) ? 2 : 1);
  if (num_arcs > 0) {
    keys_from_arcs<<<blocks_for(num_arcs), 256, 0, st>>>(
        src, dst, num_arcs, num_vertices, (flags & GB_CSR_DROP_SELF) != 0,
        (flags & GB_CSR_SYMMETRIZE) != 0, sentinel, keys);
    GB_CHECK_LAUNCH();
  }
  return keys_to_csr(keys, n, end_bit, num_vertices, sentinel, b, xadj, adj, num_edges_out, st);
}

GB_API int gb_csr_densify_workspace(int64_t num_vertices, size_t *bytes) {
  GB_REQUIRE(num_vertices >= 1 && bytes, "gb_csr_densify_workspace: bad args");
  Carver c(nullptr);
  c.take<int64_t>(num_vertices + 1);
  c.take<int64_t>(num_vertices + 1);
  c.take<int64_t>(1);
  size_t scan_bytes = 0;
  GB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int64_t *)nullptr,
                                            (int64_t *)nullptr, num_vertices + 1));
  c.take_bytes(scan_bytes);
  *bytes = c.off + 256;
  return GB_OK;
}

GB_API int gb_csr_densify(int64_t num_vertices, int64_t num_edges, const int64_t *xadj,
                              const int32_t *adj, int64_t *xadj_out, int32_t *adj_out,
                              int64_t *new_id, int64_t *kept, int64_t *num_kept_out,
                              void *workspace, size_t ws_bytes, void *stream_handle) {
  GB_REQUIRE(num_vertices >= 1 && num_edges >= 0 && xadj && xadj_out && new_id && kept &&
                 num_kept_out,
             "gb_csr_densify: bad args");
  cudaStream_t st = as_stream(stream_handle);
  Carver c(workspace);
  int64_t *flag = c.take<int64_t>(num_vertices + 1);
  int64_t *pos = c.take<int64_t>(num_vertices + 1);
  int64_t *cnt = c.take<int64_t>(1);
  size_t scan_bytes = 0;
  GB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, flag, pos, num_vertices + 1));
  void *tmp = c.take_bytes(scan_bytes);
  GB_REQUIRE(c.off <= ws_bytes, "gb_csr_densify: workspace too small");
  GB_CUDA_TRY(cudaMemsetAsync(flag + num_vertices, 0, sizeof(int64_t), st));
  nonisolated_flags<<<blocks_for(num_vertices), 256, 0, st>>>(xadj, num_vertices, flag);
  GB_CHECK_LAUNCH();
  GB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, flag, pos, num_vertices + 1, st));
  densify_vertices<<<blocks_for(num_vertices), 256, 0, st>>>(xadj, pos, num_vertices, new_id,
                                                              kept, xadj_out);
  GB_CHECK_LAUNCH();
  GB_CUDA_TRY(cudaMemcpyAsync(cnt, pos + num_vertices, sizeof(int64_t), cudaMemcpyDeviceToDevice,
                              st));
  set_tail<<<1, 1, 0, st>>>(xadj_out, cnt, num_edges);
  GB_CHECK_LAUNCH();
  if (num_edges > 0) {
    remap_adj<<<blocks_for(num_edges), 256, 0, st>>>(adj, num_edges, new_id, adj_out);
    GB_CHECK_LAUNCH();
  }
  int64_t nk = 0;
  GB_CUDA_TRY(cudaMemcpyAsync(&nk, cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA_TRY(cudaStreamSynchronize(st));
  *num_kept_out = nk;
  return GB_OK;
}

GB_API int gb_rmat_permutation_workspace(int scale, size_t *bytes) {
  GB_REQUIRE(scale >= 1 && scale <= 34 && bytes, "gb_rmat_permutation_workspace: bad args");
  const int64_t n = int64_t(1) << scale;
  Carver c(nullptr);
  c.take<uint64_t>(n);
  c.take<uint64_t>(n);
  c.take<int64_t>(n);
  size_t sb = 0;
  GB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, sb, (uint64_t *)nullptr,
                                              (uint64_t *)nullptr, (int64_t *)nullptr,
                                              (int64_t *)nullptr, n));
  c.take_bytes(sb);
  *bytes = c.off + 256;
  return GB_OK;
}

GB_API int gb_rmat_permutation(int scale, uint64_t seed, int64_t *perm, void *workspace,
                                   size_t ws_bytes, void *stream_handle) {
  GB_REQUIRE(scale >= 1 && scale <= 34 && perm, "gb_rmat_permutation: bad args");
  const int64_t n = int64_t(1) << scale;
  cudaStream_t st = as_stream(stream_handle);
  Carver c(workspace);
  uint64_t *k0 = c.take<uint64_t>(n);
  uint64_t *k1 = c.take<uint64_t>(n);
  int64_t *ids = c.take<int64_t>(n);
  size_t sb = 0;
  GB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, sb, k0, k1, ids, perm, n));
  void *tmp = c.take_bytes(sb);
  GB_REQUIRE(c.off <= ws_bytes, "gb_rmat_permutation: workspace too small");
  perm_keys<<<blocks_for(n), 256, 0, st>>>(n, stream_key(seed, kPermStream, 0, 0), k0, ids);
  GB_CHECK_LAUNCH();
  GB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, sb, k0, k1, ids, perm, n, 0, 64, st));
  return GB_OK;
}

GB_API int gb_rmat_edges(int scale, int64_t num_samples, double t_a, double t_ab,
                             double t_abc, uint64_t seed, const int64_t *perm, int64_t *src,
                             int64_t *dst, void *stream_handle) {
  GB_REQUIRE(scale >= 1 && scale <= 34 && num_samples >= 0 && src && dst,
             "gb_rmat_edges: bad args");
  if (num_samples == 0) return GB_OK;
  rmat_kernel<<<blocks_for(num_samples), 256, 0, as_stream(stream_handle)>>>(
      scale, num_samples, t_a, t_ab, t_abc, seed, perm, src, dst);
  GB_CHECK_LAUNCH();
  return GB_OK;
}

static int degree_order_layout(Carver &c, int64_t V, uint64_t **deg, uint64_t **deg_alt,
                               int64_t **ids, uint64_t **maxdeg, void **tmp, size_t *tb) {
  *deg = c.take<uint64_t>(V);
  *deg_alt = c.take<uint64_t>(V);
  *ids = c.take<int64_t>(V);
  *maxdeg = c.take<uint64_t>(1);
  size_t s1 = 0, s2 = 0;
  GB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, s1, (uint64_t *)nullptr,
                                              (uint64_t *)nullptr, (int64_t *)nullptr,
                                              (int64_t *)nullptr, V));
  GB_CUDA_TRY(cub::DeviceReduce::Max(nullptr, s2, (uint64_t *)nullptr, (uint64_t *)nullptr, V));
  *tb = std::max(s1, s2);
  *tmp = c.take_bytes(*tb);
  return GB_OK;
}

GB_API int gb_degree_order_workspace(int64_t num_vertices, size_t *bytes) {
  GB_REQUIRE(num_vertices >= 1 && bytes, "gb_degree_order_workspace: bad args");
  Carver c(nullptr);
  uint64_t *a, *b, *m;
  int64_t *ids;
  void *tmp;
  size_t tb;
  int rc = degree_order_layout(c, num_vertices, &a, &b, &ids, &m, &tmp, &tb);
  if (rc) return rc;
  *bytes = c.off + 256;
  return GB_OK;
}

GB_API int gb_degree_order(int64_t num_vertices, const int64_t *xadj, int64_t *order,
                               void *workspace, size_t ws_bytes, void *stream_handle) {
  GB_REQUIRE(num_vertices >= 1 && xadj && order, "gb_degree_order: bad args");
  cudaStream_t st = as_stream(stream_handle);
  Carver c(workspace);
  uint64_t *deg, *deg_alt, *maxdeg;
  int64_t *ids;
  void *tmp;
  size_t tb;
  int rc = degree_order_layout(c, num_vertices, &deg, &deg_alt, &ids, &maxdeg, &tmp, &tb);
  if (rc) return rc;
  GB_REQUIRE(c.off <= ws_bytes, "gb_degree_order: workspace too small");
  degrees_kernel<<<blocks_for(num_vertices), 256, 0, st>>>(xadj, num_vertices, deg, ids);
  GB_CHECK_LAUNCH();
  size_t t1 = tb;
  GB_CUDA_TRY(cub::DeviceReduce::Max(tmp, t1, deg, maxdeg, num_vertices, st));
  invert_degree_keys<<<blocks_for(num_vertices), 256, 0, st>>>(deg, num_vertices, maxdeg);
  GB_CHECK_LAUNCH();
  // stable LSD radix sort: ties (equal degree) keep ascending id order
  t1 = tb;
  GB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, t1, deg, deg_alt, ids, order, num_vertices, 0,
                                              64, st));
  return GB_OK;
}

static int collapse_layout(Carver &c, int64_t V, int64_t **rank, int8_t **status,
                           int64_t **flag, int64_t **cid, unsigned long long **undecided,
                           void **tmp, size_t *tb) {
  *rank = c.take<int64_t>(V);
  *status = c.take<int8_t>(V);
  *flag = c.take<int64_t>(V + 1);
  *cid = c.take<int64_t>(V + 1);
  *undecided = c.take<unsigned long long>(1);
  *tb = 0;
  GB_CUDA_TRY(
      cub::DeviceScan::ExclusiveSum(nullptr, *tb, (int64_t *)nullptr, (int64_t *)nullptr, V + 1));
  *tmp = c.take_bytes(*tb);
  return GB_OK;
}

GB_API int gb_collapse_workspace(int64_t num_vertices, size_t *bytes) {
  GB_REQUIRE(num_vertices >= 1 && bytes, "gb_collapse_workspace: bad args");
  Carver c(nullptr);
  int64_t *r, *f, *cid;
  int8_t *s;
  unsigned long long *u;
  void *tmp;
  size_t tb;
  int rc = collapse_layout(c, num_vertices, &r, &s, &f, &cid, &u, &tmp, &tb);
  if (rc) return rc;
  *bytes = c.off + 256;
  return GB_OK;
}

GB_API int gb_collapse(int64_t num_vertices, const int64_t *xadj, const int64_t *in_xadj,
                           const int32_t *in_adj, const int64_t *order, double delta, int32_t *cmap,
                           int64_t *num_clusters_out, int *rounds_out, void *workspace,
                           size_t ws_bytes, void *stream_handle) {
  GB_REQUIRE(num_vertices >= 1 && xadj && in_xadj && order && cmap && num_clusters_out,
             "gb_collapse: bad args");
  const int64_t V = num_vertices;
  cudaStream_t st = as_stream(stream_handle);
  Carver c(workspace);
  int64_t *rank, *flag, *cid;
  int8_t *status;
  unsigned long long *undecided;
  void *tmp;
  size_t tb;
  int rc = collapse_layout(c, V, &rank, &status, &flag, &cid, &undecided, &tmp, &tb);
  if (rc) return rc;
  GB_REQUIRE(c.off <= ws_bytes, "gb_collapse: workspace too small");
  collapse_init<<<blocks_for(V), 256, 0, st>>>(xadj, order, V, delta, rank, status);
  GB_CHECK_LAUNCH();
  const int kMaxRounds = 24;
  int rounds = 0;
  unsigned long long left = 1;
  while (left > 0 && rounds < kMaxRounds) {
    GB_CUDA_TRY(cudaMemsetAsync(undecided, 0, sizeof(unsigned long long), st));
    collapse_round<<<blocks_for(V), 256, 0, st>>>(in_xadj, in_adj, rank, V, status, undecided);
    GB_CHECK_LAUNCH();
    GB_CUDA_TRY(
        cudaMemcpyAsync(&left, undecided, sizeof(left), cudaMemcpyDeviceToHost, st));
    GB_CUDA_TRY(cudaStreamSynchronize(st));
    ++rounds;
  }
  if (left > 0) {
    collapse_tail<<<1, 32, 0, st>>>(in_xadj, in_adj, rank, order, V, status);
    GB_CHECK_LAUNCH();
    ++rounds;
  }
  GB_CUDA_TRY(cudaMemsetAsync(flag + V, 0, sizeof(int64_t), st));
  hub_flags_by_rank<<<blocks_for(V), 256, 0, st>>>(order, status, V, flag);
  GB_CHECK_LAUNCH();
  GB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, flag, cid, V + 1, st));
  assign_clusters<<<blocks_for(V), 256, 0, st>>>(in_xadj, in_adj, rank, status, cid, V, cmap);
  GB_CHECK_LAUNCH();
  int64_t nc = 0;
  GB_CUDA_TRY(cudaMemcpyAsync(&nc, cid + V, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA_TRY(cudaStreamSynchronize(st));
  *num_clusters_out = nc;
  if (rounds_out) *rounds_out = rounds;
  return GB_OK;
}

static int coarse_layout(Carver &c, int64_t E, int64_t nc, uint64_t **keys, KeyCsrBuffers &b,
                         int *end_bit, uint64_t *sentinel) {
  *sentinel = (uint64_t)nc * (uint64_t)nc;
  *end_bit = bits_for(*sentinel);
  *keys = c.take<uint64_t>(E);
  return key_csr_carve(c, E, *end_bit, b);
}

GB_API int gb_coarse_csr_workspace(int64_t num_vertices, int64_t num_edges,
                                       int64_t num_clusters, size_t *bytes) {
  GB_REQUIRE(num_vertices >= 1 && num_edges >= 0 && num_clusters >= 1 && bytes,
             "gb_coarse_csr_workspace: bad args");
  Carver c(nullptr);
  uint64_t *keys;
  KeyCsrBuffers b;
  int eb;
  uint64_t sent;
  int rc = coarse_layout(c, num_edges, num_clusters, &keys, b, &eb, &sent);
  if (rc) return rc;
  *bytes = c.off + 256;
  return GB_OK;
}

GB_API int gb_coarse_csr(int64_t num_vertices, int64_t num_edges, const int64_t *xadj,
                             const int32_t *adj, const int32_t *cmap, int64_t num_clusters,
                             int64_t *xadj_out, int32_t *adj_out, int64_t *num_edges_out,
                             void *workspace, size_t ws_bytes, void *stream_handle) {
  GB_REQUIRE(num_vertices >= 1 && num_edges >= 0 && num_clusters >= 1 && xadj && cmap &&
                 xadj_out && num_edges_out,
             "gb_coarse_csr: bad args");
  cudaStream_t st = as_stream(stream_handle);
  Carver c(workspace);
  uint64_t *keys;
  KeyCsrBuffers b;
  int end_bit;
  uint64_t sentinel;
  int rc = coarse_layout(c, num_edges, num_clusters, &keys, b, &end_bit, &sentinel);
  if (rc) return rc;
  GB_REQUIRE(c.off <= ws_bytes, "gb_coarse_csr: workspace too small");
  if (num_edges > 0) {
    int blocks = (int)std::min<int64_t>((num_vertices + 7) / 8, (int64_t)num_sms() * 16);
    coarse_keys<<<std::max(blocks, 1), 256, 0, st>>>(xadj, adj, cmap, num_vertices,
                                                     (uint64_t)num_clusters, sentinel, keys);
    GB_CHECK_LAUNCH();
  }
  return keys_to_csr(keys, num_edges, end_bit, num_clusters, sentinel, b, xadj_out, adj_out,
                     num_edges_out, st);
}

GB_API int gb_expand(const float *coarse, int64_t num_clusters, int dim, const int32_t *cmap,
                         int64_t num_rows, float *out, void *stream_handle) {
  GB_REQUIRE(coarse && cmap && out && dim >= 1 && num_rows >= 0 && num_clusters >= 1,
             "gb_expand: bad args");
  if (num_rows == 0) return GB_OK;
  cudaStream_t st = as_stream(stream_handle);
  const bool vec = dim % 4 == 0 && (reinterpret_cast<uintptr_t>(coarse) & 15u) == 0 &&
                   (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
  if (vec) {
    const int q = dim / 4;
    expand_vec4<<<blocks_for(num_rows * q), 256, 0, st>>>(
        reinterpret_cast<const float4 *>(coarse), cmap, num_rows, q,
        reinterpret_cast<float4 *>(out));
  } else {
    expand_scalar<<<blocks_for(num_rows * dim), 256, 0, st>>>(coarse, cmap, num_rows, dim, out);
  }
  GB_CHECK_LAUNCH();
  return GB_OK;
}

// Position-keyed checksum of an integer array: sum over i of
// mix64((i * GOLDEN) ^ (uint64)(int64)x[i]) mod 2^64 (elements sign-extended
// to 64 bits).  Order-sensitive through the index, associative through the
// sum, so it is one HBM pass; the oracle (or_checksum) computes the same
// number on the host.  Used to compare hierarchies whose arrays are too big
// to ship as fixtures (config-scale coarsening parity).
template <typename T>
__global__ void checksum_kernel(const T *__restrict__ x, int64_t n,
                                unsigned long long *__restrict__ out) {
  uint64_t acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc += mix64(((uint64_t)i * kGolden) ^ (uint64_t)(int64_t)__ldg(x + i));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)acc);
}

static int active_layout(Carver &c, int64_t V, int32_t **ids, char **flag, int64_t **cnt,
                         void **tmp, size_t *tb) {
  *ids = c.take<int32_t>(V);
  *flag = c.take<char>(V);
  *cnt = c.take<int64_t>(1);
  *tb = 0;
  GB_CUDA_TRY(cub::DeviceSelect::Flagged(nullptr, *tb, (int32_t *)nullptr, (char *)nullptr,
                                         (int32_t *)nullptr, (int64_t *)nullptr, V));
  *tmp = c.take_bytes(*tb);
  return GB_OK;
}

GB_API int gb_active_sources_workspace(int64_t num_vertices, size_t *bytes) {
  GB_REQUIRE(num_vertices >= 1 && num_vertices < (int64_t(1) << 31) && bytes,
             "gb_active_sources_workspace: bad args");
  Carver c(nullptr);
  int32_t *ids;
  char *flag;
  int64_t *cnt;
  void *tmp;
  size_t tb;
  int rc = active_layout(c, num_vertices, &ids, &flag, &cnt, &tmp, &tb);
  if (rc) return rc;
  *bytes = c.off + 256;
  return GB_OK;
}

GB_API int gb_active_sources(int64_t num_vertices, const int64_t *xadj, int32_t *out,
                             int64_t *count_out, void *workspace, size_t ws_bytes,
                             void *stream_handle) {
  GB_REQUIRE(num_vertices >= 1 && xadj && out && count_out, "gb_active_sources: bad args");
  cudaStream_t st = as_stream(stream_handle);
  Carver c(workspace);
  int32_t *ids;
  char *flag;
  int64_t *cnt;
  void *tmp;
  size_t tb;
  int rc = active_layout(c, num_vertices, &ids, &flag, &cnt, &tmp, &tb);
  if (rc) return rc;
  GB_REQUIRE(c.off <= ws_bytes, "gb_active_sources: workspace too small");
  active_flags<<<blocks_for(num_vertices), 256, 0, st>>>(xadj, num_vertices, ids, flag);
  GB_CHECK_LAUNCH();
  GB_CUDA_TRY(cub::DeviceSelect::Flagged(tmp, tb, ids, flag, out, cnt, num_vertices, st));
  int64_t n = 0;
  GB_CUDA_TRY(cudaMemcpyAsync(&n, cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA_TRY(cudaStreamSynchronize(st));
  *count_out = n;
  return GB_OK;
}

GB_API int gb_checksum(const void *data, int64_t n, int elem_bytes, uint64_t *out,
                       void *stream_handle) {
  GB_REQUIRE(out && n >= 0 && (n == 0 || data), "gb_checksum: bad args");
  GB_REQUIRE(elem_bytes == 4 || elem_bytes == 8, "gb_checksum: elem_bytes must be 4 or 8");
  cudaStream_t st = as_stream(stream_handle);
  GB_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(uint64_t), st));
  if (n == 0) return GB_OK;
  const int grid = (int)std::min<int64_t>(blocks_for(n), (int64_t)num_sms() * 8);
  auto *o = reinterpret_cast<unsigned long long *>(out);
  if (elem_bytes == 4)
    checksum_kernel<<<grid, 256, 0, st>>>(static_cast<const int32_t *>(data), n, o);
  else
    checksum_kernel<<<grid, 256, 0, st>>>(static_cast<const int64_t *>(data), n, o);
  GB_CHECK_LAUNCH();
  return GB_OK;
}

// ---------------------------------------------------------------------------
// Row-block (chunked) CSR construction.  The one-shot builds above hold the
// keys of every arc three times over (keys, sorted copy, unique copy: 24 B
// per arc, ~190 GB for C5's 8B arcs); here only one block of source rows
// [r0, r1) is keyed, sorted and emitted at a time, so the scratch scales
// with the block.  The host picks blocks from a per-source arc histogram
// (an upper bound: duplicates are counted until the block's unique pass)
// and streams the arcs through in batches (device arc arrays, R-MAT sample
// batches, or a CSR mapped through a cluster map for the coarse graph).
// Blocks emit rows in order, so the concatenated output is the one-shot
// build's CSR bit for bit.
// ---------------------------------------------------------------------------
__global__ void arc_hist_kernel(const int64_t *__restrict__ src, const int64_t *__restrict__ dst,
                                int64_t n, bool drop_self, bool sym,
                                unsigned long long *__restrict__ hist) {
  GRID_STRIDE(i, n) {
    const int64_t s = src[i], d = dst[i];
    if (drop_self && s == d) continue;
    atomicAdd(hist + s, 1ull);
    if (sym) atomicAdd(hist + d, 1ull);
  }
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// keys (s - r0) * V + d of the arcs whose source lies in [r0, r1), appended
// at a warp-aggregated cursor (order inside the block is irrelevant: sorted next)
__global__ void arc_keys_range_kernel(const int64_t *__restrict__ src,
                                      const int64_t *__restrict__ dst, int64_t n, bool drop_self,
                                      bool sym, int64_t r0, int64_t r1, uint64_t V,
                                      uint64_t *__restrict__ keys,
                                      unsigned long long *__restrict__ cursor) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < n;
       i0 += stride) {
    const int64_t i = i0 + lane;
    bool e1 = false, e2 = false;
    uint64_t k1 = 0, k2 = 0;
    if (i < n) {
      const int64_t s = src[i], d = dst[i];
      if (!(drop_self && s == d)) {
        if (s >= r0 && s < r1) {
          e1 = true;
          k1 = (uint64_t)(s - r0) * V + (uint64_t)d;
        }
        if (sym && d >= r0 && d < r1) {
          e2 = true;
          k2 = (uint64_t)(d - r0) * V + (uint64_t)s;
        }
      }
    }
    const unsigned m1 = __ballot_sync(0xffffffffu, e1), m2 = __ballot_sync(0xffffffffu, e2);
    const int tot = __popc(m1) + __popc(m2);
    if (tot == 0) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(cursor, (unsigned long long)tot);
    base = __shfl_sync(0xffffffffu, base, 0);
    const unsigned lt = lanemask_lt();
    if (e1) keys[base + __popc(m1 & lt)] = k1;
    if (e2) keys[base + __popc(m1) + __popc(m2 & lt)] = k2;
  }
}

// coarse arcs (cmap[v], cmap[u]) of a CSR, intra-cluster arcs dropped
// (coarsen.py:200-253): per-cluster histogram, warp per vertex
__global__ void mapped_hist_kernel(const int64_t *__restrict__ xadj,
                                   const int32_t *__restrict__ adj,
                                   const int32_t *__restrict__ cmap, int64_t V,
                                   unsigned long long *__restrict__ hist) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < V; v += nwarps) {
    const int32_t cv = cmap[v];
    unsigned cnt = 0;
    for (int64_t e = xadj[v] + lane; e < xadj[v + 1]; e += 32) cnt += cmap[adj[e]] != cv;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    if (lane == 0 && cnt) atomicAdd(hist + cv, (unsigned long long)cnt);
  }
}

__global__ void mapped_keys_range_kernel(const int64_t *__restrict__ xadj,
                                         const int32_t *__restrict__ adj,
                                         const int32_t *__restrict__ cmap, int64_t V, int64_t c0,
                                         int64_t c1, uint64_t nc, uint64_t *__restrict__ keys,
                                         unsigned long long *__restrict__ cursor) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned lt = lanemask_lt();
  for (int64_t v = warp; v < V; v += nwarps) {
    const int64_t cv = cmap[v];
    if (cv < c0 || cv >= c1) continue;  // warp-uniform
    const int64_t e0 = xadj[v], e1 = xadj[v + 1];
    for (int64_t eb = e0; eb < e1; eb += 32) {
      const int64_t e = eb + lane;
      int64_t cu = cv;
      if (e < e1) cu = cmap[adj[e]];
      const bool emit = cu != cv;
      const unsigned m = __ballot_sync(0xffffffffu, emit);
      if (!m) continue;
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(cursor, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (emit) keys[base + __popc(m & lt)] = (uint64_t)(cv - c0) * nc + (uint64_t)cu;
    }
  }
}

// Same keys as mapped_keys_range_kernel, appended per ROW: row_cursor[r]
// (r = cluster - c0) starts at the row's offset in the block's key buffer (an
// exclusive scan of gb_mapped_histogram over the block) and ends at the next
// row's.  The single block-wide cursor serialised every 32-key append on one
// L2 address (~60 ms per 1G keys at the C5 shape); per-row cursors spread
// them over the block's rows.  Each warp tests the clusters of 32 of its
// vertices at once (warp w owns vertices w, w + nwarps, ...: the hubs, which
// lead the rank-ordered ids of a coarse level, stay spread over the warps).
// the contracted arcs e0..e1 of a vertex of cluster cv, appended by one warp
__device__ __forceinline__ void append_mapped_arcs(const int32_t *__restrict__ adj,
                                                   const int32_t *__restrict__ cmap,
                                                   int64_t e0, int64_t e1, int64_t cv,
                                                   int64_t c0, uint64_t nc,
                                                   uint64_t *__restrict__ keys,
                                                   unsigned long long *__restrict__ row_cursor,
                                                   int lane, unsigned lt) {
  for (int64_t eb = e0; eb < e1; eb += 32) {
    const int64_t e = eb + lane;
    int64_t cu = cv;
    if (e < e1) cu = cmap[adj[e]];
    const bool emit = cu != cv;
    const unsigned m = __ballot_sync(0xffffffffu, emit);
    if (!m) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(row_cursor + (cv - c0), (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (emit) keys[base + __popc(m & lt)] = (uint64_t)(cv - c0) * nc + (uint64_t)cu;
  }
}

// Vertices with more than heavy_arcs arcs (the hubs of a coarse level: one
// warp walking a 10M-arc hub held a whole block's launch for ~130 ms at C5)
// are queued instead and split into kHeavyPieces pieces for all warps
// (mapped_keys_rows_heavy_kernel); a full queue falls back to the warp.
constexpr int64_t kHeavyPieces = 64;

__global__ void mapped_keys_rows_kernel(const int64_t *__restrict__ xadj,
                                        const int32_t *__restrict__ adj,
                                        const int32_t *__restrict__ cmap, int64_t V, int64_t c0,
                                        int64_t c1, uint64_t nc, uint64_t *__restrict__ keys,
                                        unsigned long long *__restrict__ row_cursor,
                                        int64_t *__restrict__ heavy, int64_t heavy_cap,
                                        int64_t heavy_arcs,
                                        unsigned long long *__restrict__ heavy_count) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned lt = lanemask_lt();
  for (int64_t vb = warp; vb < V; vb += nwarps * 32) {
    const int64_t vl = vb + (int64_t)lane * nwarps;
    const int32_t cl = vl < V ? cmap[vl] : -1;
    unsigned in_range = __ballot_sync(0xffffffffu, vl < V && cl >= c0 && cl < c1);
    while (in_range) {
      const int src_lane = __ffs(in_range) - 1;
      in_range &= in_range - 1;
      const int64_t v = vb + (int64_t)src_lane * nwarps;
      const int64_t cv = __shfl_sync(0xffffffffu, cl, src_lane);
      const int64_t e0 = xadj[v], e1 = xadj[v + 1];
      if (heavy_cap > 0 && e1 - e0 > heavy_arcs) {
        unsigned long long slot = 0;
        if (lane == 0) slot = atomicAdd(heavy_count, 1ull);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if ((int64_t)slot < heavy_cap) {
          if (lane == 0) heavy[slot] = v;
          continue;
        }
      }
      append_mapped_arcs(adj, cmap, e0, e1, cv, c0, nc, keys, row_cursor, lane, lt);
    }
  }
}

__global__ void mapped_keys_rows_heavy_kernel(const int64_t *__restrict__ xadj,
                                              const int32_t *__restrict__ adj,
                                              const int32_t *__restrict__ cmap, int64_t c0,
                                              uint64_t nc, uint64_t *__restrict__ keys,
                                              unsigned long long *__restrict__ row_cursor,
                                              const int64_t *__restrict__ heavy,
                                              int64_t heavy_cap,
                                              const unsigned long long *__restrict__ heavy_count) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned lt = lanemask_lt();
  const int64_t queued = (int64_t)*heavy_count, n = queued < heavy_cap ? queued : heavy_cap;
  for (int64_t item = warp; item < n * kHeavyPieces; item += nwarps) {
    const int64_t v = heavy[item / kHeavyPieces], piece = item % kHeavyPieces;
    const int64_t e0 = xadj[v], e1 = xadj[v + 1];
    const int64_t len = ((e1 - e0 + kHeavyPieces - 1) / kHeavyPieces + 31) & ~int64_t(31);
    const int64_t a = e0 + piece * len, b = e1 < a + len ? e1 : a + len;
    if (a >= b) continue;
    append_mapped_arcs(adj, cmap, a, b, (int64_t)cmap[v], c0, nc, keys, row_cursor, lane, lt);
  }
}

// rows [r0, r1) of xadj from the block's sorted unique keys (row-relative)
__global__ void xadj_rows_from_keys(const uint64_t *__restrict__ keys, int64_t nkeys,
                                    int64_t rows, uint64_t ncols, int64_t base,
                                    int64_t *__restrict__ xadj_rows) {
  GRID_STRIDE(r, rows) {
    const uint64_t target = (uint64_t)r * ncols;
    int64_t lo = 0, hi = nkeys;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target)
        lo = mid + 1;
      else
        hi = mid;
    }
    xadj_rows[r] = base + lo;
  }
}

GB_API int gb_arc_histogram(const int64_t *src, const int64_t *dst, int64_t num_arcs,
                            unsigned flags, int64_t *hist, void *stream_handle) {
  GB_REQUIRE(num_arcs >= 0 && hist && (num_arcs == 0 || (src && dst)),
             "gb_arc_histogram: bad args");
  if (num_arcs == 0) return GB_OK;
  arc_hist_kernel<<<blocks_for(num_arcs), 256, 0, as_stream(stream_handle)>>>(
      src, dst, num_arcs, flags & GB_CSR_DROP_SELF, flags & GB_CSR_SYMMETRIZE,
      reinterpret_cast<unsigned long long *>(hist));
  GB_CHECK_LAUNCH();
  return GB_OK;
}

GB_API int gb_arc_keys_range(const int64_t *src, const int64_t *dst, int64_t num_arcs,
                             unsigned flags, int64_t num_vertices, int64_t r0, int64_t r1,
                             uint64_t *keys, int64_t *cursor, void *stream_handle) {
  GB_REQUIRE(num_arcs >= 0 && keys && cursor && r0 >= 0 && r1 >= r0 && r1 <= num_vertices,
             "gb_arc_keys_range: bad args");
  if (num_arcs == 0 || r1 == r0) return GB_OK;
  arc_keys_range_kernel<<<blocks_for(num_arcs), 256, 0, as_stream(stream_handle)>>>(
      src, dst, num_arcs, flags & GB_CSR_DROP_SELF, flags & GB_CSR_SYMMETRIZE, r0, r1,
      (uint64_t)num_vertices, keys, reinterpret_cast<unsigned long long *>(cursor));
  GB_CHECK_LAUNCH();
  return GB_OK;
}

GB_API int gb_mapped_histogram(const int64_t *xadj, const int32_t *adj, int64_t num_vertices,
                               const int32_t *cmap, int64_t *hist, void *stream_handle) {
  GB_REQUIRE(num_vertices >= 1 && xadj && cmap && hist, "gb_mapped_histogram: bad args");
  const int blocks = (int)std::min<int64_t>((num_vertices + 7) / 8, (int64_t)num_sms() * 16);
  mapped_hist_kernel<<<std::max(blocks, 1), 256, 0, as_stream(stream_handle)>>>(
      xadj, adj, cmap, num_vertices, reinterpret_cast<unsigned long long *>(hist));
  GB_CHECK_LAUNCH();
  return GB_OK;
}

GB_API int gb_mapped_keys_range(const int64_t *xadj, const int32_t *adj, int64_t num_vertices,
                                const int32_t *cmap, int64_t num_clusters, int64_t c0,
                                int64_t c1, uint64_t *keys, int64_t *cursor,
                                void *stream_handle) {
  GB_REQUIRE(num_vertices >= 1 && xadj && cmap && keys && cursor && c0 >= 0 && c1 >= c0 &&
                 c1 <= num_clusters,
             "gb_mapped_keys_range: bad args");
  if (c1 == c0) return GB_OK;
  const int blocks = (int)std::min<int64_t>((num_vertices + 7) / 8, (int64_t)num_sms() * 16);
  mapped_keys_range_kernel<<<std::max(blocks, 1), 256, 0, as_stream(stream_handle)>>>(
      xadj, adj, cmap, num_vertices, c0, c1, (uint64_t)num_clusters, keys,
      reinterpret_cast<unsigned long long *>(cursor));
  GB_CHECK_LAUNCH();
  return GB_OK;
}

GB_API int gb_mapped_keys_rows(const int64_t *xadj, const int32_t *adj, int64_t num_vertices,
                               const int32_t *cmap, int64_t num_clusters, int64_t c0,
                               int64_t c1, int64_t *row_cursor, uint64_t *keys,
                               int64_t *heavy, int64_t heavy_cap, int64_t heavy_arcs,
                               void *stream_handle) {
  GB_REQUIRE(num_vertices >= 1 && xadj && cmap && keys && row_cursor && c0 >= 0 && c1 >= c0 &&
                 c1 <= num_clusters && heavy_cap >= 0 && (heavy_cap == 0 || heavy) &&
                 heavy_arcs >= 32,
             "gb_mapped_keys_rows: bad args");
  if (c1 == c0) return GB_OK;
  cudaStream_t st = as_stream(stream_handle);
  // heavy[0] counts the queue, heavy[1..heavy_cap] holds it
  unsigned long long *count = reinterpret_cast<unsigned long long *>(heavy);
  if (heavy_cap > 0) GB_CUDA_TRY(cudaMemsetAsync(heavy, 0, sizeof(int64_t), st));
  const int blocks =
      (int)std::min<int64_t>((num_vertices + 255) / 256, (int64_t)num_sms() * 16);
  mapped_keys_rows_kernel<<<std::max(blocks, 1), 256, 0, st>>>(
      xadj, adj, cmap, num_vertices, c0, c1, (uint64_t)num_clusters, keys,
      reinterpret_cast<unsigned long long *>(row_cursor), heavy_cap ? heavy + 1 : nullptr,
      heavy_cap, heavy_arcs, count);
  GB_CHECK_LAUNCH();
  if (heavy_cap > 0) {
    mapped_keys_rows_heavy_kernel<<<num_sms() * 8, 256, 0, st>>>(
        xadj, adj, cmap, c0, (uint64_t)num_clusters, keys,
        reinterpret_cast<unsigned long long *>(row_cursor), heavy + 1, heavy_cap, count);
    GB_CHECK_LAUNCH();
  }
  return GB_OK;
}

GB_API int gb_keys_to_rows_workspace(int64_t num_keys, int64_t rows, int64_t num_cols,
                                     size_t *bytes) {
  GB_REQUIRE(num_keys >= 0 && rows >= 1 && num_cols >= 1 && bytes,
             "gb_keys_to_rows_workspace: bad args");
  Carver c(nullptr);
  KeyCsrBuffers b;
  int rc = key_csr_carve(c, std::max<int64_t>(num_keys, 1),
                         bits_for((uint64_t)rows * (uint64_t)num_cols), b);
  if (rc) return rc;
  *bytes = c.off + 256;
  return GB_OK;
}

// Sort + deduplicate one block's keys and emit its rows: xadj_rows[0..rows)
// (offset by `base`, the arcs of the earlier blocks) and adj_out[0..unique).
// Synchronizes; *num_unique_out (host) sizes the next block's offset.
GB_API int gb_keys_to_rows(uint64_t *keys, int64_t num_keys, int64_t rows, int64_t num_cols,
                           int64_t base, int64_t *xadj_rows, int32_t *adj_out,
                           int64_t *num_unique_out, void *workspace, size_t ws_bytes,
                           void *stream_handle) {
  GB_REQUIRE(num_keys >= 0 && rows >= 1 && num_cols >= 1 && xadj_rows && num_unique_out &&
                 (num_keys == 0 || (keys && adj_out)),
             "gb_keys_to_rows: bad args");
  cudaStream_t st = as_stream(stream_handle);
  Carver c(workspace);
  KeyCsrBuffers b;
  const int end_bit = bits_for((uint64_t)rows * (uint64_t)num_cols);
  int rc = key_csr_carve(c, std::max<int64_t>(num_keys, 1), end_bit, b);
  if (rc) return rc;
  GB_REQUIRE(c.off <= ws_bytes, "gb_keys_to_rows: workspace too small");
  int64_t nuniq = 0;
  if (num_keys > 0) {
    size_t tb = b.cub_bytes;
    GB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(b.cub_tmp, tb, keys, b.keys_alt, num_keys, 0,
                                               end_bit, st));
    tb = b.cub_bytes;
    GB_CUDA_TRY(
        cub::DeviceSelect::Unique(b.cub_tmp, tb, b.keys_alt, b.uniq, b.num_sel, num_keys, st));
    GB_CUDA_TRY(cudaMemcpyAsync(&nuniq, b.num_sel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GB_CUDA_TRY(cudaStreamSynchronize(st));
  }
  xadj_rows_from_keys<<<blocks_for(rows), 256, 0, st>>>(b.uniq, nuniq, rows,
                                                         (uint64_t)num_cols, base, xadj_rows);
  GB_CHECK_LAUNCH();
  if (nuniq > 0) {
    adj_from_keys<<<blocks_for(nuniq), 256, 0, st>>>(b.uniq, nuniq, num_cols, adj_out);
    GB_CHECK_LAUNCH();
  }
  GB_CUDA_TRY(cudaStreamSynchronize(st));
  *num_unique_out = nuniq;
  return GB_OK;
}

GB_API int gb_rmat_edges_range(int scale, int64_t first, int64_t count, double t_a, double t_ab,
                               double t_abc, uint64_t seed, const int64_t *perm, int64_t *src,
                               int64_t *dst, void *stream_handle) {
  GB_REQUIRE(scale >= 1 && scale <= 34 && first >= 0 && count >= 0 && src && dst,
             "gb_rmat_edges_range: bad args");
  if (count == 0) return GB_OK;
  rmat_range_kernel<<<blocks_for(count), 256, 0, as_stream(stream_handle)>>>(
      scale, first, count, t_a, t_ab, t_abc, seed, perm, src, dst);
  GB_CHECK_LAUNCH();
  return GB_OK;
}

// ---------------------------------------------------------------------------
// Run-dependent parallel collapse (coarsen.py:117-179 _collapse_par +
// _normalize): the reference's try-lock/skip-on-failure mode, not part of the
// parity contract.  A worker is one warp: it grabs kGrab consecutive order
// positions from a shared cursor (GRAB_BATCH, coarsen.py:30), claims each
// vertex as a hub with a CAS (provisional cluster id = its own id) and
// offers its eligible neighbours to the hub with a CAS each (the lanes take
// the row 32 arcs at a time: distinct u, so lane order is irrelevant); a
// lost CAS skips the vertex, as the reference does.  One worker reproduces
// the sequential collapse exactly; more workers give a valid map that
// depends on the interleaving.  Normalisation numbers hubs by their order
// position (flag + exclusive scan), like _normalize.
// ---------------------------------------------------------------------------
static constexpr int kGrab = 64;  // coarsen.py:30 GRAB_BATCH

__global__ void collapse_cas_kernel(const int64_t *__restrict__ xadj,
                                    const int32_t *__restrict__ adj,
                                    const int64_t *__restrict__ order, int64_t V, double delta,
                                    int32_t *cmap, unsigned long long *cursor) {
  const int lane = threadIdx.x & 31;
  volatile int32_t *vmap = cmap;
  for (;;) {
    unsigned long long lo = 0;
    if (lane == 0) lo = atomicAdd(cursor, (unsigned long long)kGrab);
    lo = __shfl_sync(0xffffffffu, lo, 0);
    if ((int64_t)lo >= V) break;
    const int64_t hi = min((int64_t)lo + kGrab, V);
    for (int64_t i = (int64_t)lo; i < hi; ++i) {
      const int64_t v = order[i];
      int claimed = 0;
      if (lane == 0) claimed = atomicCAS(cmap + v, -1, (int32_t)v) == -1;
      if (!__shfl_sync(0xffffffffu, claimed, 0)) continue;
      const int64_t b = xadj[v], e = xadj[v + 1];
      const bool v_small = (double)(e - b) <= delta;  // coarsen.py:108
      for (int64_t k = b + lane; k < e; k += 32) {
        const int32_t u = adj[k];
        if (vmap[u] != -1) continue;
        if (v_small || (double)(xadj[u + 1] - xadj[u]) <= delta)  // coarsen.py:111
          atomicCAS(cmap + u, -1, (int32_t)v);
      }
      __syncwarp();
    }
  }
}

__global__ void cas_hub_flags(const int64_t *__restrict__ order, const int32_t *__restrict__ cmap,
                              int64_t V, int64_t *__restrict__ flag) {
  GRID_STRIDE(i, V) {
    const int64_t v = order[i];
    flag[i] = cmap[v] == (int32_t)v ? 1 : 0;
  }
}

__global__ void cas_dense_ids(const int64_t *__restrict__ order, const int64_t *__restrict__ flag,
                              const int64_t *__restrict__ cid, int64_t V,
                              int32_t *__restrict__ dense) {
  GRID_STRIDE(i, V) if (flag[i]) dense[order[i]] = (int32_t)cid[i];
}

__global__ void cas_normalize(const int32_t *__restrict__ prov, const int32_t *__restrict__ dense,
                              int64_t V, int32_t *__restrict__ out) {
  GRID_STRIDE(v, V) out[v] = dense[prov[v]];
}

static int collapse_cas_layout(Carver &c, int64_t V, unsigned long long **cursor, int32_t **prov,
                        int32_t **dense, int64_t **flag, int64_t **cid, void **tmp,
                        size_t *tb) {
  *cursor = c.take<unsigned long long>(1);
  *prov = c.take<int32_t>(V);
  *dense = c.take<int32_t>(V);
  *flag = c.take<int64_t>(V + 1);
  *cid = c.take<int64_t>(V + 1);
  *tb = 0;
  GB_CUDA_TRY(
      cub::DeviceScan::ExclusiveSum(nullptr, *tb, (int64_t *)nullptr, (int64_t *)nullptr, V + 1));
  *tmp = c.take_bytes(*tb);
  return GB_OK;
}
GB_API int gb_collapse_cas_workspace(int64_t num_vertices, size_t *bytes) {
  GB_REQUIRE(num_vertices >= 1 && num_vertices < (int64_t)INT32_MAX && bytes,
             "gb_collapse_cas_workspace: bad args");
  Carver c(nullptr);
  unsigned long long *cur;
  int32_t *p, *d;
  int64_t *f, *cid;
  void *tmp;
  size_t tb;
  int rc = collapse_cas_layout(c, num_vertices, &cur, &p, &d, &f, &cid, &tmp, &tb);
  if (rc) return rc;
  *bytes = c.off + 256;
  return GB_OK;
}

GB_API int gb_collapse_cas(int64_t num_vertices, const int64_t *xadj, const int32_t *adj,
                           const int64_t *order, double delta, int64_t num_workers,
                           int32_t *cmap, int64_t *num_clusters_out, void *workspace,
                           size_t ws_bytes, void *stream_handle) {
  GB_REQUIRE(num_vertices >= 1 && num_vertices < (int64_t)INT32_MAX && xadj && adj && order &&
                 cmap && num_clusters_out && num_workers >= 1,
             "gb_collapse_cas: bad args");
  const int64_t V = num_vertices;
  cudaStream_t st = as_stream(stream_handle);
  Carver c(workspace);
  unsigned long long *cursor;
  int32_t *prov, *dense;
  int64_t *flag, *cid;
  void *tmp;
  size_t tb;
  int rc = collapse_cas_layout(c, V, &cursor, &prov, &dense, &flag, &cid, &tmp, &tb);
  if (rc) return rc;
  GB_REQUIRE(c.off <= ws_bytes, "gb_collapse_cas: workspace too small");
  GB_CUDA_TRY(cudaMemsetAsync(prov, 0xff, V * sizeof(int32_t), st));
  GB_CUDA_TRY(cudaMemsetAsync(cursor, 0, sizeof(unsigned long long), st));
  // workers = warps; never more than there are batches to grab
  const int64_t batches = (V + kGrab - 1) / kGrab;
  const int64_t warps = std::min<int64_t>(std::min<int64_t>(num_workers, batches),
                                          (int64_t)num_sms() * 64);
  const int wpb = (int)std::min<int64_t>(warps, 8);
  const int blocks = (int)((warps + wpb - 1) / wpb);
  collapse_cas_kernel<<<blocks, wpb * 32, 0, st>>>(xadj, adj, order, V, delta, prov, cursor);
  GB_CHECK_LAUNCH();
  cas_hub_flags<<<blocks_for(V), 256, 0, st>>>(order, prov, V, flag);
  GB_CHECK_LAUNCH();
  GB_CUDA_TRY(cudaMemsetAsync(flag + V, 0, sizeof(int64_t), st));
  GB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, flag, cid, V + 1, st));
  cas_dense_ids<<<blocks_for(V), 256, 0, st>>>(order, flag, cid, V, dense);
  GB_CHECK_LAUNCH();
  cas_normalize<<<blocks_for(V), 256, 0, st>>>(prov, dense, V, cmap);
  GB_CHECK_LAUNCH();
  int64_t nc = 0;
  GB_CUDA_TRY(cudaMemcpyAsync(&nc, cid + V, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA_TRY(cudaStreamSynchronize(st));
  *num_clusters_out = nc;
  return GB_OK;
}
