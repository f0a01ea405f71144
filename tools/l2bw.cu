// l2bw.cu -- measurement tool (not part of libgsg): the on-chip ceilings that bound the SpMM
// when its gathered feature matrix is L2-resident (SURVEY §8(d) "Measure L2 read bandwidth on
// the box once ... and record it beside MEASURED_PEAKS").
//   1. streaming read of a buffer that fits in L2 (float4 loads, repeated passes)
//   2. random 512-byte row gathers from an L2-resident [rows x 128] fp32 slab (the SpMM's
//      access pattern: one warp = one 128-column chunk of one neighbor row)
//   3. streaming read of a 4 GB buffer (HBM) for reference
// Prints one JSON line. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/l2bw.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k_stream(const float4* __restrict__ p, size_t n4, int passes, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r = 0; r < passes; r++)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = __ldg(p + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) *out = acc.x;
}

// each warp: `iters` gathers of one 512-byte row chunk at a pseudo-random row, 8 in flight
__global__ void k_gather(const float4* __restrict__ slab, int rows, int ld4, int iters, float* out) {
  const int lane = threadIdx.x & 31;
  unsigned s = (blockIdx.x * blockDim.x + threadIdx.x) / 32 * 2654435761u + 12345u;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int it = 0; it < iters; it += 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      s = s * 1664525u + 1013904223u;
      v[u] = __ldg(slab + (size_t)(s % rows) * ld4 + lane);
    }
#pragma unroll
    for (int u = 0; u < 8; u++) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
  }
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) *out = acc.x;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  // 1. L2-resident streaming read (32 MB)
  size_t bytes = 32u << 20;
  float4* buf;
  cudaMalloc(&buf, (size_t)4 << 30);
  cudaMemset(buf, 0, (size_t)4 << 30);
  const int passes = 50;
  k_stream<<<sms * 8, 256>>>(buf, bytes / 16, 2, out);
  cudaEventRecord(a);
  k_stream<<<sms * 8, 256>>>(buf, bytes / 16, passes, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  double l2_stream = (double)bytes * passes / (ms / 1e3) / 1e9;
  // 2. gathers of 512-byte row chunks from a 10 MB slab (20000 rows x 128 fp32)
  const int rows = 20000, ld4 = 32, iters = 4096;
  const int blocks = sms * 8;
  k_gather<<<blocks, 256>>>(buf, rows, ld4, 64, out);
  cudaEventRecord(a);
  k_gather<<<blocks, 256>>>(buf, rows, ld4, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  double gathers = (double)blocks * 8 * iters;  // warps x iterations
  double l2_gather = gathers * 512.0 / (ms / 1e3) / 1e9;
  // 3. HBM streaming read (4 GB, one pass)
  size_t hb = (size_t)4 << 30;
  k_stream<<<sms * 8, 256>>>(buf, hb / 16, 1, out);
  cudaEventRecord(a);
  k_stream<<<sms * 8, 256>>>(buf, hb / 16, 1, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  double hbm_read = (double)hb / (ms / 1e3) / 1e9;
  printf("{\"l2_bytes\": %d, \"sms\": %d, \"l2_stream_read_gbs\": %.1f, \"l2_gather512_gbs\": %.1f, "
         "\"hbm_stream_read_gbs\": %.1f, \"err\": \"%s\"}\n",
         l2, sms, l2_stream, l2_gather, hbm_read, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
