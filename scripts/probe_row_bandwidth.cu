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
// 5 rows in flight per group (the pass's source + 4 samples).
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
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
