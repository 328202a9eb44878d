// Practical ceiling of the training pass's memory pattern on this GPU
// (measurement tool, not product code): random 512-byte row gathers followed
// by 16-byte vector-reduction write-backs of the same rows -- the pass
// kernel's traffic with no arithmetic -- against a streaming copy.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/probe_rows \
//        scripts/probe_row_bandwidth.cu && build/probe_rows
//
// Rows are float[128] (d = 128); a group of 8 lanes moves one row as 8 x 4
// float4 (the pass kernel's VecRow<8,4> layout).  Row ids are uniform over a
// 512 MiB matrix (inputs larger than L2).  Prints JSON lines with GB/s of
// algorithmic bytes (read + write per row) for: copy, gather (read only),
// gather + red.add (read-modify-write, the pass pattern), and the same with
// 5 rows in flight per group (the pass's source + 4 samples).  The "tma"
// patterns move the same rows with bulk-async copies instead
// (cp.async.bulk global->shared, one 512-byte copy per row, completion on a
// per-warp mbarrier, two stages per warp so the next item's rows are in
// flight while the current ones are consumed): does the TMA path raise the
// ceiling of random-row traffic above the LSU path?  "tma gather+bulk-reduce"
// also writes back through the TMA unit (cp.reduce.async.bulk .add.f32 of
// the row from its shared slot).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void copy_kernel(const float4 *__restrict__ a, float4 *__restrict__ b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = __ldcg(a + i);
}

// mode 0: gather only; 1: gather + red.add of the same row
template <int ROWS>
__global__ void rows_kernel(float *M, int64_t V, int64_t items, int mode, uint64_t seed,
                            float *sink) {
  const int lane = threadIdx.x & 31, gl = lane & 7;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int64_t groups = ((int64_t)gridDim.x * blockDim.x) >> 3;
  float acc = 0.f;
  for (int64_t it = group; it < items; it += groups) {
    float4 r[ROWS][4];
    int64_t id[ROWS];
#pragma unroll
    for (int j = 0; j < ROWS; ++j) {
      id[j] = (int64_t)(mix64(seed ^ (uint64_t)(it * ROWS + j)) % (uint64_t)V);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        r[j][k] = __ldcg(reinterpret_cast<const float4 *>(M + id[j] * 128) + k * 8 + gl);
    }
#pragma unroll
    for (int j = 0; j < ROWS; ++j) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc += r[j][k].x + r[j][k].y + r[j][k].z + r[j][k].w;
        if (mode == 1) {
          float *p = M + id[j] * 128 + 4 * (k * 8 + gl);
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p),
                       "f"(1e-30f), "f"(1e-30f), "f"(1e-30f), "f"(1e-30f)
                       : "memory");
        }
      }
    }
  }
  if (acc == 12345.f) sink[0] = acc;
}

// TMA variant: each warp takes 4 items (4 groups of 8 lanes, as above) per
// step; lanes 0..4*ROWS-1 each issue one 512-byte bulk copy of a row into the
// warp's stage buffer.  Consumers read the rows from shared memory (and
// red.add them back for mode 1).
template <int ROWS>
__global__ void __launch_bounds__(128) tma_rows_kernel(float *M, int64_t V, int64_t items,
                                                       int mode, uint64_t seed, float *sink) {
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t mbar[4][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, grp = lane >> 3, gl = lane & 7;
  constexpr int NR = 4 * ROWS;  // rows per warp step
  float *buf = smem + (size_t)warp * 2 * NR * 128;
  const int64_t wid = (int64_t)blockIdx.x * 4 + warp, nw = (int64_t)gridDim.x * 4;
  if (lane == 0) {
    for (int s = 0; s < 2; ++s) {
      uint32_t a = (uint32_t)__cvta_generic_to_shared(&mbar[warp][s]);
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(a));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  auto row_id = [&](int64_t step, int r) {
    const int64_t it = step * 4 + r / ROWS;
    return (int64_t)(mix64(seed ^ (uint64_t)(it * ROWS + r % ROWS)) % (uint64_t)V);
  };
  auto issue = [&](int64_t step, int s) {
    uint32_t bar = (uint32_t)__cvta_generic_to_shared(&mbar[warp][s]);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar),
                   "r"(NR * 512) : "memory");
    __syncwarp();
    if (lane < NR) {
      // mode 2: this lane's bulk reduction out of the slot must have read it
      if (mode == 2) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      const float *src = M + row_id(step, lane) * 128;
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf + ((size_t)s * NR + lane) * 128);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, "
          "[%2];" ::"r"(dst), "l"(src), "r"(bar) : "memory");
    }
  };
  const int64_t steps = items / 4;
  float acc = 0.f;
  uint32_t phase[2] = {0, 0};
  int s = 0;
  if (wid < steps) issue(wid, 0);
  for (int64_t step = wid; step < steps; step += nw) {
    if (step + nw < steps) issue(step + nw, s ^ 1);
    uint32_t bar = (uint32_t)__cvta_generic_to_shared(&mbar[warp][s]);
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done) : "r"(bar), "r"(phase[s]) : "memory");
    phase[s] ^= 1;
#pragma unroll
    for (int j = 0; j < ROWS; ++j) {
      const int r = grp * ROWS + j;
      const float4 *row = reinterpret_cast<const float4 *>(buf + ((size_t)s * NR + r) * 128);
      const int64_t id = mode ? row_id(step, r) : 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float4 v = row[k * 8 + gl];
        acc += v.x + v.y + v.z + v.w;
        if (mode == 1) {
          float *p = M + id * 128 + 4 * (k * 8 + gl);
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p),
                       "f"(1e-30f), "f"(1e-30f), "f"(1e-30f), "f"(1e-30f)
                       : "memory");
        } else if (mode == 2) {  // the delta goes back into the slot
          const_cast<float4 *>(row)[k * 8 + gl] = make_float4(1e-30f, 1e-30f, 1e-30f, 1e-30f);
        }
      }
    }
    if (mode == 2) {  // one bulk reduce-add per row, smem slot -> global row
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane < NR) {
        float *dst = M + row_id(step, lane) * 128;
        uint32_t src = (uint32_t)__cvta_generic_to_shared(buf + ((size_t)s * NR + lane) * 128);
        asm volatile(
            "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 512;"
            ::"l"(dst), "r"(src) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    __syncwarp();
    s ^= 1;
  }
  if (mode == 2 && lane < NR) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (acc == 12345.f) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t V = 1 << 20;  // 1M rows x 512 B = 512 MiB
  float *M, *B, *sink;
  cudaMalloc(&M, V * 128 * sizeof(float));
  cudaMalloc(&B, V * 128 * sizeof(float));
  cudaMalloc(&sink, 4);
  cudaMemset(M, 0, V * 128 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 10;
  };
  const int64_t n4 = V * 32;
  float ms = time([&] { copy_kernel<<<sms * 8, 256>>>((float4 *)M, (float4 *)B, n4); });
  printf("{\"pattern\": \"copy\", \"GBps\": %.1f}\n", 2.0 * V * 512 / (ms * 1e6));
  const int64_t items = 4 * V;
  for (int blocks_per_sm : {2, 3, 4, 8}) {
    for (int mode = 0; mode < 2; ++mode) {
      ms = time([&] {
        rows_kernel<1><<<sms * blocks_per_sm, 256>>>(M, V, items, mode, 7, sink);
      });
      double bytes = (double)items * 512 * (mode ? 2 : 1);
      printf("{\"pattern\": \"%s\", \"rows_in_flight_per_group\": 1, \"blocks_per_sm\": %d, "
             "\"GBps\": %.1f}\n", mode ? "gather+red" : "gather", blocks_per_sm,
             bytes / (ms * 1e6));
      ms = time([&] {
        rows_kernel<5><<<sms * blocks_per_sm, 256>>>(M, V, items / 5, mode, 9, sink);
      });
      bytes = (double)(items / 5) * 5 * 512 * (mode ? 2 : 1);
      printf("{\"pattern\": \"%s\", \"rows_in_flight_per_group\": 5, \"blocks_per_sm\": %d, "
             "\"GBps\": %.1f}\n", mode ? "gather+red" : "gather", blocks_per_sm,
             bytes / (ms * 1e6));
    }
  }
  for (int rows : {1, 5}) {
    const int smem_bytes = 4 * 2 * 4 * rows * 512;  // 4 warps x 2 stages x 4 groups x rows
    auto kern = rows == 1 ? tma_rows_kernel<1> : tma_rows_kernel<5>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, smem_bytes);
    for (int mode = 0; mode < 3; ++mode) {
      const int64_t its = items / rows;
      ms = time([&] { kern<<<sms * occ, 128, smem_bytes>>>(M, V, its, mode, 11, sink); });
      double bytes = (double)its * rows * 512 * (mode ? 2 : 1);
      printf("{\"pattern\": \"tma %s\", \"rows_in_flight_per_group\": %d, \"stages\": 2, "
             "\"blocks_per_sm\": %d, \"warps_per_sm\": %d, \"GBps\": %.1f}\n",
             mode == 2 ? "gather+bulk-reduce" : mode ? "gather+red" : "gather", rows, occ,
             occ * 4, bytes / (ms * 1e6));
    }
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
