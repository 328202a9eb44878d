// Train/test split and negative-pair membership on the device (reference:
// graph.py:46-59 undirected_pairs, graph.py:222-265 split_train_test,
// evaluate.py:80-125 sample_negative_edges), SURVEY.md 8(f) rank 3.
//
// The random choices stay numpy's (Generator(PCG64).choice / .integers on the
// host, so the selected edges and candidate pairs are identical to the
// reference's); everything O(|E|) around them runs here:
//
//   gb_undirected_pairs   arcs (u, v) with u < v in CSR order -- per-row
//                         upper bound of u in the sorted row, exclusive scan,
//                         one warp per row writing its tail
//   gb_split_partition    test flags from the chosen indices, train/test
//                         compaction, vertices kept by the train edges,
//                         dense relabel (scan), test pairs that lost an
//                         endpoint dropped
//   gb_pairs_member       (u, v) is an arc (binary search in row u) or is an
//                         excluded pair (binary search in a sorted key list)
//
// Integer/byte work, HBM-bound; grids are multiples of the SM count.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace gb {
namespace {

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
};

inline int grid_for(int64_t n, int threads = 256) {
  const int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms() * 32));
}

#define GRID_STRIDE(i, n)                                                   \
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); \
       i += (int64_t)gridDim.x * blockDim.x)

// first index in adj[lo, hi) with adj > x (rows ascending)
__device__ __forceinline__ int64_t upper_bound_row(const int32_t *__restrict__ adj, int64_t lo,
                                                   int64_t hi, int64_t x) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)__ldg(adj + mid) <= x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__global__ void tail_counts(const int64_t *__restrict__ xadj, const int32_t *__restrict__ adj,
                            int64_t V, int64_t *__restrict__ first, int64_t *__restrict__ cnt) {
  GRID_STRIDE(u, V) {
    const int64_t e1 = xadj[u + 1];
    const int64_t f = upper_bound_row(adj, xadj[u], e1, u);
    first[u] = f;
    cnt[u] = e1 - f;
  }
}

// one warp per row: pairs[off[u] + j] = (u, adj[first[u] + j])
__global__ void write_tails(const int32_t *__restrict__ adj, int64_t V,
                            const int64_t *__restrict__ first, const int64_t *__restrict__ cnt,
                            const int64_t *__restrict__ off, int64_t *__restrict__ pu,
                            int64_t *__restrict__ pv) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < V; u += warps) {
    const int64_t f = first[u], c = cnt[u], o = off[u];
    for (int64_t j = lane; j < c; j += 32) {
      pu[o + j] = u;
      pv[o + j] = __ldg(adj + f + j);
    }
  }
}

__global__ void mark_chosen(const int64_t *__restrict__ chosen, int64_t k, int64_t m,
                            uint8_t *__restrict__ is_test, int *__restrict__ bad) {
  GRID_STRIDE(i, k) {
    const int64_t c = chosen[i];
    if (c < 0 || c >= m)
      *bad = 1;
    else
      is_test[c] = 1;
  }
}

__global__ void mark_used(const int64_t *__restrict__ pu, const int64_t *__restrict__ pv,
                          const uint8_t *__restrict__ is_test, int64_t m,
                          int64_t *__restrict__ used) {
  GRID_STRIDE(i, m) {
    if (!is_test[i]) {
      used[pu[i]] = 1;  // benign same-value races
      used[pv[i]] = 1;
    }
  }
}

__global__ void kept_and_relabel(const int64_t *__restrict__ used, const int64_t *__restrict__ pos,
                                 int64_t V, int64_t *__restrict__ relabel,
                                 int64_t *__restrict__ kept) {
  GRID_STRIDE(u, V) {
    if (used[u]) {
      relabel[u] = pos[u];
      kept[pos[u]] = u;
    } else {
      relabel[u] = -1;
    }
  }
}

// train pairs (relabelled) and test pairs (relabelled, both endpoints kept)
// into flagged compaction inputs
__global__ void relabel_pairs(const int64_t *__restrict__ pu, const int64_t *__restrict__ pv,
                              const uint8_t *__restrict__ is_test, int64_t m,
                              const int64_t *__restrict__ relabel, int64_t *__restrict__ ru,
                              int64_t *__restrict__ rv, uint8_t *__restrict__ train_flag,
                              uint8_t *__restrict__ test_flag) {
  GRID_STRIDE(i, m) {
    const int64_t a = relabel[pu[i]], b = relabel[pv[i]];
    ru[i] = a;
    rv[i] = b;
    const bool t = is_test[i];
    train_flag[i] = !t;
    test_flag[i] = t && a >= 0 && b >= 0;
  }
}

__global__ void pairs_member_kernel(const int64_t *__restrict__ xadj,
                                    const int32_t *__restrict__ adj, int64_t V,
                                    const int64_t *__restrict__ u, const int64_t *__restrict__ v,
                                    int64_t n, const int64_t *__restrict__ excl, int64_t n_excl,
                                    uint8_t *__restrict__ out) {
  GRID_STRIDE(i, n) {
    const int64_t a = u[i], b = v[i];
    bool hit = false;
    if (a >= 0 && a < V) {
      const int64_t e0 = xadj[a], e1 = xadj[a + 1];
      const int64_t p = upper_bound_row(adj, e0, e1, b - 1);  // first adj >= b
      hit = p < e1 && (int64_t)__ldg(adj + p) == b;
    }
    if (!hit && n_excl > 0) {
      const int64_t key = a * V + b;
      int64_t lo = 0, hi = n_excl;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (excl[mid] < key)
          lo = mid + 1;
        else
          hi = mid;
      }
      hit = lo < n_excl && excl[lo] == key;
    }
    out[i] = hit ? 1 : 0;
  }
}

__global__ void excl_keys(const int64_t *__restrict__ eu, const int64_t *__restrict__ ev,
                          int64_t n, int64_t V, int64_t *__restrict__ keys) {
  GRID_STRIDE(i, n) {
    keys[i] = eu[i] * V + ev[i];
    keys[n + i] = ev[i] * V + eu[i];
  }
}

}  // namespace
}  // namespace gb

using namespace gb;

// ---- undirected_pairs -----------------------------------------------------------
static int pairs_layout(Carver &c, int64_t V, int64_t **first, int64_t **cnt, int64_t **off,
                        void **tmp, size_t *tmp_bytes) {
  *first = c.take<int64_t>(V);
  *cnt = c.take<int64_t>(V + 1);
  *off = c.take<int64_t>(V + 1);
  size_t b = 0;
  GB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, b, (int64_t *)nullptr, (int64_t *)nullptr,
                                            V + 1));
  *tmp = c.take<char>(b);
  *tmp_bytes = b;
  return GB_OK;
}

GB_API int gb_undirected_pairs_workspace(int64_t num_vertices, size_t *bytes) {
  GB_REQUIRE(num_vertices >= 1 && bytes, "gb_undirected_pairs_workspace: bad args");
  Carver c(nullptr);
  int64_t *f, *n, *o;
  void *t;
  size_t tb;
  int rc = pairs_layout(c, num_vertices, &f, &n, &o, &t, &tb);
  if (rc) return rc;
  *bytes = c.off + 256;
  return GB_OK;
}

GB_API int gb_undirected_pairs(const int64_t *xadj, const int32_t *adj, int64_t num_vertices,
                               int64_t *pu, int64_t *pv, int64_t capacity, int64_t *num_pairs,
                               void *workspace, size_t ws_bytes, void *stream) {
  GB_REQUIRE(xadj && num_pairs && workspace && num_vertices >= 1,
             "gb_undirected_pairs: bad args");
  cudaStream_t st = as_stream(stream);
  Carver c(workspace);
  int64_t *first, *cnt, *off;
  void *tmp;
  size_t tb;
  int rc = pairs_layout(c, num_vertices, &first, &cnt, &off, &tmp, &tb);
  if (rc) return rc;
  GB_REQUIRE(c.off <= ws_bytes, "gb_undirected_pairs: workspace too small");
  tail_counts<<<grid_for(num_vertices), 256, 0, st>>>(xadj, adj, num_vertices, first, cnt);
  GB_CHECK_LAUNCH();
  GB_CUDA_TRY(cudaMemsetAsync(cnt + num_vertices, 0, sizeof(int64_t), st));
  GB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, num_vertices + 1, st));
  int64_t m = 0;
  GB_CUDA_TRY(cudaMemcpyAsync(&m, off + num_vertices, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA_TRY(cudaStreamSynchronize(st));
  *num_pairs = m;
  GB_REQUIRE(m <= capacity, "gb_undirected_pairs: %lld pairs exceed capacity %lld",
             (long long)m, (long long)capacity);
  if (m > 0) {
    GB_REQUIRE(pu && pv, "gb_undirected_pairs: null output");
    write_tails<<<grid_for(num_vertices * 32), 256, 0, st>>>(adj, num_vertices, first, cnt, off,
                                                             pu, pv);
    GB_CHECK_LAUNCH();
  }
  return GB_OK;
}

// ---- split partition --------------------------------------------------------------
struct SplitBufs {
  uint8_t *is_test, *train_flag, *test_flag;
  int64_t *used, *pos, *ru, *rv, *nsel;
  int *bad;
  void *tmp;
  size_t tmp_bytes;
};

static int split_layout(Carver &c, int64_t m, int64_t V, SplitBufs &b) {
  b.is_test = c.take<uint8_t>(m);
  b.train_flag = c.take<uint8_t>(m);
  b.test_flag = c.take<uint8_t>(m);
  b.used = c.take<int64_t>(V + 1);
  b.pos = c.take<int64_t>(V + 1);
  b.ru = c.take<int64_t>(m);
  b.rv = c.take<int64_t>(m);
  b.nsel = c.take<int64_t>(4);
  b.bad = c.take<int>(1);
  size_t s1 = 0, s2 = 0;
  GB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, s1, (int64_t *)nullptr, (int64_t *)nullptr,
                                            V + 1));
  GB_CUDA_TRY(cub::DeviceSelect::Flagged(nullptr, s2, (int64_t *)nullptr, (uint8_t *)nullptr,
                                         (int64_t *)nullptr, (int64_t *)nullptr, m));
  b.tmp_bytes = std::max(s1, s2);
  b.tmp = c.take<char>(b.tmp_bytes);
  return GB_OK;
}

GB_API int gb_split_partition_workspace(int64_t num_pairs, int64_t num_vertices, size_t *bytes) {
  GB_REQUIRE(num_pairs >= 0 && num_vertices >= 1 && bytes,
             "gb_split_partition_workspace: bad args");
  Carver c(nullptr);
  SplitBufs b;
  int rc = split_layout(c, num_pairs, num_vertices, b);
  if (rc) return rc;
  *bytes = c.off + 256;
  return GB_OK;
}

// counts[0] = train pairs, counts[1] = surviving test pairs, counts[2] = kept
// vertices (host memory; the call synchronizes the stream).
GB_API int gb_split_partition(const int64_t *pu, const int64_t *pv, int64_t num_pairs,
                              const int64_t *chosen, int64_t k, int64_t num_vertices,
                              int64_t *train_u, int64_t *train_v, int64_t *test_u,
                              int64_t *test_v, int64_t *relabel, int64_t *kept, int64_t *counts,
                              void *workspace, size_t ws_bytes, void *stream) {
  GB_REQUIRE(pu && pv && num_pairs >= 1 && num_vertices >= 1 && counts && workspace,
             "gb_split_partition: bad args");
  GB_REQUIRE(k == 0 || chosen, "gb_split_partition: null chosen");
  GB_REQUIRE(train_u && train_v && test_u && test_v && relabel && kept,
             "gb_split_partition: null output");
  cudaStream_t st = as_stream(stream);
  Carver c(workspace);
  SplitBufs b;
  int rc = split_layout(c, num_pairs, num_vertices, b);
  if (rc) return rc;
  GB_REQUIRE(c.off <= ws_bytes, "gb_split_partition: workspace too small");
  const int64_t m = num_pairs, V = num_vertices;
  GB_CUDA_TRY(cudaMemsetAsync(b.is_test, 0, m, st));
  GB_CUDA_TRY(cudaMemsetAsync(b.used, 0, sizeof(int64_t) * (V + 1), st));
  GB_CUDA_TRY(cudaMemsetAsync(b.bad, 0, sizeof(int), st));
  if (k > 0) {
    mark_chosen<<<grid_for(k), 256, 0, st>>>(chosen, k, m, b.is_test, b.bad);
    GB_CHECK_LAUNCH();
  }
  mark_used<<<grid_for(m), 256, 0, st>>>(pu, pv, b.is_test, m, b.used);
  GB_CHECK_LAUNCH();
  GB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(b.tmp, b.tmp_bytes, b.used, b.pos, V + 1, st));
  kept_and_relabel<<<grid_for(V), 256, 0, st>>>(b.used, b.pos, V, relabel, kept);
  GB_CHECK_LAUNCH();
  relabel_pairs<<<grid_for(m), 256, 0, st>>>(pu, pv, b.is_test, m, relabel, b.ru, b.rv,
                                             b.train_flag, b.test_flag);
  GB_CHECK_LAUNCH();
  size_t tb = b.tmp_bytes;
  GB_CUDA_TRY(cub::DeviceSelect::Flagged(b.tmp, tb, b.ru, b.train_flag, train_u, b.nsel, m, st));
  GB_CUDA_TRY(cub::DeviceSelect::Flagged(b.tmp, tb, b.rv, b.train_flag, train_v, b.nsel, m, st));
  GB_CUDA_TRY(
      cub::DeviceSelect::Flagged(b.tmp, tb, b.ru, b.test_flag, test_u, b.nsel + 1, m, st));
  GB_CUDA_TRY(
      cub::DeviceSelect::Flagged(b.tmp, tb, b.rv, b.test_flag, test_v, b.nsel + 1, m, st));
  int64_t h[3];
  int bad = 0;
  GB_CUDA_TRY(cudaMemcpyAsync(h, b.nsel, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA_TRY(cudaMemcpyAsync(h + 2, b.pos + V, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA_TRY(cudaMemcpyAsync(&bad, b.bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  GB_CUDA_TRY(cudaStreamSynchronize(st));
  GB_REQUIRE(!bad, "gb_split_partition: chosen index out of range");
  counts[0] = h[0];
  counts[1] = h[1];
  counts[2] = h[2];
  return GB_OK;
}

// ---- pair membership ----------------------------------------------------------------
GB_API int gb_pairs_member_workspace(int64_t num_excluded, size_t *bytes) {
  GB_REQUIRE(num_excluded >= 0 && bytes, "gb_pairs_member_workspace: bad args");
  Carver c(nullptr);
  const int64_t n2 = 2 * num_excluded;
  c.take<int64_t>(n2);
  c.take<int64_t>(n2);
  size_t sb = 0;
  if (n2 > 0)
    GB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, sb, (int64_t *)nullptr,
                                               (int64_t *)nullptr, n2));
  c.take<char>(sb);
  *bytes = c.off + 256;
  return GB_OK;
}

// out[i] = 1 iff (u[i], v[i]) is an arc of the CSR or (u, v) / (v, u) is one
// of the excluded pairs (evaluate.py:97-119).
GB_API int gb_pairs_member(const int64_t *xadj, const int32_t *adj, int64_t num_vertices,
                           const int64_t *u, const int64_t *v, int64_t n,
                           const int64_t *excl_u, const int64_t *excl_v, int64_t num_excluded,
                           uint8_t *out, void *workspace, size_t ws_bytes, void *stream) {
  GB_REQUIRE(xadj && num_vertices >= 1 && n >= 0, "gb_pairs_member: bad args");
  if (n == 0) return GB_OK;
  GB_REQUIRE(u && v && out, "gb_pairs_member: null pointer");
  cudaStream_t st = as_stream(stream);
  const int64_t n2 = 2 * num_excluded;
  int64_t *sorted = nullptr;
  if (n2 > 0) {
    GB_REQUIRE(excl_u && excl_v && workspace, "gb_pairs_member: null excluded pairs");
    Carver c(workspace);
    int64_t *keys = c.take<int64_t>(n2);
    sorted = c.take<int64_t>(n2);
    size_t sb = 0;
    GB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, sb, keys, sorted, n2));
    void *tmp = c.take<char>(sb);
    GB_REQUIRE(c.off <= ws_bytes, "gb_pairs_member: workspace too small");
    excl_keys<<<grid_for(num_excluded), 256, 0, st>>>(excl_u, excl_v, num_excluded, num_vertices,
                                                      keys);
    GB_CHECK_LAUNCH();
    GB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp, sb, keys, sorted, n2, 0, 64, st));
  }
  pairs_member_kernel<<<grid_for(n), 256, 0, st>>>(xadj, adj, num_vertices, u, v, n, sorted, n2,
                                                   out);
  GB_CHECK_LAUNCH();
  return GB_OK;
}
