// Graph input on the device: the GSHG loader's
// validation (graph.py:61-77 Graph.validate, called by load_graph,
// graph.py:203-219) and the text edge-list parser (graph.py:134-171
// load_edge_list) with its id densification.
//
// Byte work bounded by HBM: validation reads xadj and adj once (a row-start
// bitmap turns the per-row "strictly ascending" rule into a coalesced
// per-arc test); the parser reads each text byte about twice (line starts,
// then one thread per line) and writes 16 B per edge.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

using namespace gb;

namespace {

struct Carve {
  char *base;
  size_t off = 0;
  explicit Carve(void *b) : base(static_cast<char *>(b)) {}
  template <class T>
  T *take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
};

inline int grid_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms() * 32));
}

#define STRIDE(i, n)                                                        \
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); \
       i += (int64_t)gridDim.x * blockDim.x)

// ---------------------------------------------------------------------------
// CSR validation.  flags bits (the reference's checks, in its order):
//   1 xadj endpoints (xadj[0] != 0 or xadj[V] != E)
//   2 xadj decreasing somewhere
//   4 adj entry out of [0, V)
//   8 a row not strictly ascending (only meaningful when 1 and 2 are clear)
// ---------------------------------------------------------------------------
__global__ void validate_rows(const int64_t *__restrict__ xadj, int64_t V, int64_t E,
                              unsigned *__restrict__ starts, int *__restrict__ flags) {
  int f = 0;
  STRIDE(v, V) {
    const int64_t a = xadj[v], b = xadj[v + 1];
    if (b < a) f |= 2;
    // a nonempty row starting inside [1, E) marks a boundary
    if (v > 0 && a < b && a > 0 && a < E) atomicOr(starts + (a >> 5), 1u << (a & 31));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (xadj[0] != 0 || xadj[V] != E)) f |= 1;
  if (f) atomicOr(flags, f);
}

__global__ void validate_arcs(const int32_t *__restrict__ adj, int64_t V, int64_t E,
                              const unsigned *__restrict__ starts, int *__restrict__ flags) {
  int f = 0;
  STRIDE(e, E) {
    const int32_t x = adj[e];
    if (x < 0 || (int64_t)x >= V) f |= 4;
    if (e > 0 && !((starts[e >> 5] >> (e & 31)) & 1u) && x <= adj[e - 1]) f |= 8;
  }
  if (f) atomicOr(flags, f);
}

// ---------------------------------------------------------------------------
// Edge-list text.  A line ends at '\n' (text streams hand over universal-
// newline-translated text); whitespace is str.isspace's ASCII set.  Status
// per line: 0 edge, 1 skipped (blank or '#' after leading whitespace),
// 2 parse error (field count or a field int() rejects), 3 both ids valid
// Python ints but one outside int64 (numpy's conversion raises later).
// int() syntax: [+-]? digit (_? digit)*  (base 10, leading zeros allowed).
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool is_ws(unsigned char c) {
  return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f);
}

// 0 ok, 2 syntax error, 3 overflow
__device__ int parse_int(const unsigned char *s, int64_t n, int64_t *out) {
  int64_t i = 0;
  bool neg = false;
  if (i < n && (s[i] == '+' || s[i] == '-')) {
    neg = s[i] == '-';
    ++i;
  }
  if (i >= n) return 2;
  unsigned long long mag = 0;
  bool over = false, prev_digit = false;
  for (; i < n; ++i) {
    const unsigned char c = s[i];
    if (c >= '0' && c <= '9') {
      const unsigned d = c - '0';
      if (mag > (~0ull - d) / 10ull) over = true;
      else mag = mag * 10ull + d;
      prev_digit = true;
    } else if (c == '_') {
      if (!prev_digit || i + 1 >= n || s[i + 1] < '0' || s[i + 1] > '9') return 2;
      prev_digit = false;
    } else {
      return 2;
    }
  }
  if (!prev_digit) return 2;
  const unsigned long long lim = neg ? (1ull << 63) : ((1ull << 63) - 1);
  if (over || mag > lim) return 3;
  *out = neg ? (int64_t)(0ull - mag) : (int64_t)mag;
  return 0;
}

// Also flags text the host must parse: a byte >= 0x80 (int() accepts
// non-ASCII digits and str.split non-ASCII spaces) or a '\r' not followed by
// '\n' (a line break under universal newlines).
__global__ void line_start_flags(const unsigned char *__restrict__ text, int64_t n,
                                 uint8_t *__restrict__ flag, int *__restrict__ needs_host) {
  int h = 0;
  STRIDE(p, n) {
    const unsigned char c = text[p];
    flag[p] = (p == 0 || text[p - 1] == '\n') ? 1 : 0;
    if (c >= 0x80 || (c == '\r' && (p + 1 >= n || text[p + 1] != '\n'))) h = 1;
  }
  if (h) atomicOr(needs_host, 1);
}

__global__ void parse_lines(const unsigned char *__restrict__ text, int64_t n,
                            const int64_t *__restrict__ starts, int64_t L,
                            int64_t *__restrict__ U, int64_t *__restrict__ Vv,
                            uint8_t *__restrict__ ok, unsigned long long *__restrict__ first_bad,
                            int *__restrict__ any_overflow) {
  STRIDE(i, L) {
    int64_t p = starts[i];
    const int64_t end_hint = (i + 1 < L) ? starts[i + 1] : n;
    int64_t e = end_hint;
    if (e > p && text[e - 1] == '\n') --e;
    while (p < e && is_ws(text[p])) ++p;
    while (e > p && is_ws(text[e - 1])) --e;
    int status = 1;
    if (p < e && text[p] != '#') {
      // split on whitespace runs; keep the first two fields
      int64_t fb[2] = {0, 0}, fe[2] = {0, 0};
      int fields = 0;
      int64_t q = p;
      while (q < e) {
        while (q < e && is_ws(text[q])) ++q;
        if (q >= e) break;
        const int64_t b = q;
        while (q < e && !is_ws(text[q])) ++q;
        if (fields < 2) {
          fb[fields] = b;
          fe[fields] = q;
        }
        ++fields;
      }
      if (fields != 2) {
        status = 2;
      } else {
        int64_t u = 0, v = 0;
        const int su = parse_int(text + fb[0], fe[0] - fb[0], &u);
        const int sv = parse_int(text + fb[1], fe[1] - fb[1], &v);
        if (su == 2 || sv == 2) {
          status = 2;
        } else if (su == 3 || sv == 3) {
          status = 3;
        } else {
          status = 0;
          U[i] = u;
          Vv[i] = v;
        }
      }
    }
    // overflowing lines still count as edges (the reference appends them and
    // fails at the int64 conversion after the loop)
    ok[i] = status == 0 ? 1 : 0;
    if (status == 2) atomicMin(first_bad, (unsigned long long)i);
    if (status == 3) atomicOr(any_overflow, 1);
  }
}

__global__ void lower_bound_ids(const int64_t *__restrict__ sorted, int64_t n_sorted,
                                int64_t *__restrict__ ids, int64_t n) {
  STRIDE(i, n) {
    const int64_t x = ids[i];
    int64_t lo = 0, hi = n_sorted;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (sorted[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    ids[i] = lo;
  }
}

struct TextLayout {
  uint8_t *flag;
  int64_t *starts, *U, *V, *nsel;
  uint8_t *ok;
  unsigned long long *first_bad;
  int *overflow;
  int *needs_host;
  void *tmp;
  size_t tmp_bytes;
};

int text_layout(Carve &c, int64_t n, TextLayout &t) {
  t.flag = c.take<uint8_t>(n);
  t.starts = c.take<int64_t>(n);
  t.U = c.take<int64_t>(n);
  t.V = c.take<int64_t>(n);
  t.ok = c.take<uint8_t>(n);
  t.nsel = c.take<int64_t>(1);
  t.first_bad = c.take<unsigned long long>(1);
  t.overflow = c.take<int>(1);
  t.needs_host = c.take<int>(1);
  size_t a = 0, b = 0;
  thrust::counting_iterator<int64_t> it(0);
  GB_CUDA_TRY(cub::DeviceSelect::Flagged(nullptr, a, it, (uint8_t *)nullptr, (int64_t *)nullptr,
                                         (int64_t *)nullptr, n));
  GB_CUDA_TRY(cub::DeviceSelect::Flagged(nullptr, b, (int64_t *)nullptr, (uint8_t *)nullptr,
                                         (int64_t *)nullptr, (int64_t *)nullptr, n));
  t.tmp_bytes = std::max(a, b);
  t.tmp = c.take<char>(t.tmp_bytes);
  return GB_OK;
}

}  // namespace

GB_API int gb_csr_validate_workspace(int64_t num_edges, size_t *bytes) {
  GB_REQUIRE(num_edges >= 0 && bytes, "gb_csr_validate_workspace: bad args");
  *bytes = (size_t)((num_edges + 31) / 32 + 1) * sizeof(unsigned) + sizeof(int) + 512;
  return GB_OK;
}

GB_API int gb_csr_validate(int64_t num_vertices, int64_t num_edges, const int64_t *xadj,
                           const int32_t *adj, int *flags_out, void *workspace,
                           size_t ws_bytes, void *stream_handle) {
  GB_REQUIRE(num_vertices >= 0 && num_edges >= 0 && xadj && (adj || num_edges == 0) &&
                 flags_out,
             "gb_csr_validate: bad args");
  cudaStream_t st = as_stream(stream_handle);
  Carve c(workspace);
  const int64_t words = (num_edges + 31) / 32 + 1;
  unsigned *starts = c.take<unsigned>(words);
  int *flags = c.take<int>(1);
  GB_REQUIRE(c.off <= ws_bytes, "gb_csr_validate: workspace too small");
  GB_CUDA_TRY(cudaMemsetAsync(starts, 0, words * sizeof(unsigned), st));
  GB_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(int), st));
  validate_rows<<<grid_for(std::max<int64_t>(num_vertices, 1)), 256, 0, st>>>(
      xadj, num_vertices, num_edges, starts, flags);
  GB_CHECK_LAUNCH();
  if (num_edges > 0) {
    validate_arcs<<<grid_for(num_edges), 256, 0, st>>>(adj, num_vertices, num_edges, starts,
                                                       flags);
    GB_CHECK_LAUNCH();
  }
  GB_CUDA_TRY(cudaMemcpyAsync(flags_out, flags, sizeof(int), cudaMemcpyDeviceToHost, st));
  GB_CUDA_TRY(cudaStreamSynchronize(st));
  return GB_OK;
}

GB_API int gb_parse_edge_text_workspace(int64_t num_bytes, size_t *bytes) {
  GB_REQUIRE(num_bytes >= 1 && bytes, "gb_parse_edge_text_workspace: bad args");
  Carve c(nullptr);
  TextLayout t;
  int rc = text_layout(c, num_bytes, t);
  if (rc) return rc;
  *bytes = c.off + 256;
  return GB_OK;
}

GB_API int gb_parse_edge_text(const char *text, int64_t num_bytes, int64_t *u_out,
                              int64_t *v_out, int64_t *result, void *workspace,
                              size_t ws_bytes, void *stream_handle) {
  GB_REQUIRE(text && num_bytes >= 1 && u_out && v_out && result,
             "gb_parse_edge_text: bad args");
  cudaStream_t st = as_stream(stream_handle);
  Carve c(workspace);
  TextLayout t;
  int rc = text_layout(c, num_bytes, t);
  if (rc) return rc;
  GB_REQUIRE(c.off <= ws_bytes, "gb_parse_edge_text: workspace too small");
  const unsigned char *s = reinterpret_cast<const unsigned char *>(text);
  GB_CUDA_TRY(cudaMemsetAsync(t.needs_host, 0, sizeof(int), st));
  line_start_flags<<<grid_for(num_bytes), 256, 0, st>>>(s, num_bytes, t.flag, t.needs_host);
  GB_CHECK_LAUNCH();
  thrust::counting_iterator<int64_t> it(0);
  size_t tb = t.tmp_bytes;
  GB_CUDA_TRY(cub::DeviceSelect::Flagged(t.tmp, tb, it, t.flag, t.starts, t.nsel, num_bytes, st));
  int64_t L = 0;
  GB_CUDA_TRY(cudaMemcpyAsync(&L, t.nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA_TRY(cudaMemsetAsync(t.first_bad, 0xff, sizeof(unsigned long long), st));
  GB_CUDA_TRY(cudaMemsetAsync(t.overflow, 0, sizeof(int), st));
  GB_CUDA_TRY(cudaStreamSynchronize(st));
  parse_lines<<<grid_for(L), 256, 0, st>>>(s, num_bytes, t.starts, L, t.U, t.V, t.ok,
                                           t.first_bad, t.overflow);
  GB_CHECK_LAUNCH();
  tb = t.tmp_bytes;
  GB_CUDA_TRY(cub::DeviceSelect::Flagged(t.tmp, tb, t.U, t.ok, u_out, t.nsel, L, st));
  tb = t.tmp_bytes;
  GB_CUDA_TRY(cub::DeviceSelect::Flagged(t.tmp, tb, t.V, t.ok, v_out, t.nsel, L, st));
  int64_t m = 0;
  unsigned long long bad = 0;
  int over = 0, host = 0;
  GB_CUDA_TRY(cudaMemcpyAsync(&m, t.nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA_TRY(cudaMemcpyAsync(&bad, t.first_bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
  GB_CUDA_TRY(cudaMemcpyAsync(&over, t.overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
  GB_CUDA_TRY(cudaMemcpyAsync(&host, t.needs_host, sizeof(int), cudaMemcpyDeviceToHost, st));
  GB_CUDA_TRY(cudaStreamSynchronize(st));
  result[0] = m;
  result[1] = L;
  result[2] = bad == ~0ull ? -1 : (int64_t)bad;
  result[3] = over;
  result[4] = host;
  return GB_OK;
}

GB_API int gb_unique_ids_workspace(int64_t n, size_t *bytes) {
  GB_REQUIRE(n >= 1 && bytes, "gb_unique_ids_workspace: bad args");
  size_t a = 0, b = 0;
  GB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, a, (int64_t *)nullptr, (int64_t *)nullptr,
                                             n));
  GB_CUDA_TRY(cub::DeviceSelect::Unique(nullptr, b, (int64_t *)nullptr, (int64_t *)nullptr,
                                        (int64_t *)nullptr, n));
  Carve c(nullptr);
  c.take<int64_t>(n);
  c.take<int64_t>(1);
  c.take<char>(std::max(a, b));
  *bytes = c.off + 256;
  return GB_OK;
}

// Sorted distinct values of ids[0..n) into uniq (n entries of room); then,
// with relabel set, every ids[i] is replaced by its rank in uniq
// (np.unique + np.searchsorted, graph.py:160-164).
GB_API int gb_unique_ids(int64_t *ids, int64_t n, int64_t *uniq, int64_t *num_unique_out,
                         int relabel, void *workspace, size_t ws_bytes, void *stream_handle) {
  GB_REQUIRE(ids && uniq && num_unique_out && n >= 1, "gb_unique_ids: bad args");
  cudaStream_t st = as_stream(stream_handle);
  size_t a = 0, b = 0;
  GB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, a, (int64_t *)nullptr, (int64_t *)nullptr,
                                             n));
  GB_CUDA_TRY(cub::DeviceSelect::Unique(nullptr, b, (int64_t *)nullptr, (int64_t *)nullptr,
                                        (int64_t *)nullptr, n));
  Carve c(workspace);
  int64_t *sorted = c.take<int64_t>(n);
  int64_t *nsel = c.take<int64_t>(1);
  size_t tb = std::max(a, b);
  void *tmp = c.take<char>(tb);
  GB_REQUIRE(c.off <= ws_bytes, "gb_unique_ids: workspace too small");
  size_t t1 = tb;
  GB_CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp, t1, ids, sorted, n, 0, 64, st));
  t1 = tb;
  GB_CUDA_TRY(cub::DeviceSelect::Unique(tmp, t1, sorted, uniq, nsel, n, st));
  int64_t k = 0;
  GB_CUDA_TRY(cudaMemcpyAsync(&k, nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GB_CUDA_TRY(cudaStreamSynchronize(st));
  if (relabel) {
    lower_bound_ids<<<grid_for(n), 256, 0, st>>>(uniq, k, ids, n);
    GB_CHECK_LAUNCH();
  }
  *num_unique_out = k;
  return GB_OK;
}
