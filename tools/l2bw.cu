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

// each warp: `iters` gathers of a (W x 512)-byte row chunk at a pseudo-random row; U rows in flight
template <int W, int U>
__global__ void k_gather(const float4* __restrict__ slab, int rows, int ld4, int iters, float* out) {
  const int lane = threadIdx.x & 31;
  unsigned s = (blockIdx.x * blockDim.x + threadIdx.x) / 32 * 2654435761u + 12345u;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int it = 0; it < iters; it += U) {
    float4 v[U][W];
#pragma unroll
    for (int u = 0; u < U; u++) {
      s = s * 1664525u + 1013904223u;
#pragma unroll
      for (int w = 0; w < W; w++) v[u][w] = __ldg(slab + (size_t)(s % rows) * ld4 + lane + 32 * w);
    }
#pragma unroll
    for (int u = 0; u < U; u++)
#pragma unroll
      for (int w = 0; w < W; w++) { acc.x += v[u][w].x; acc.y += v[u][w].y; acc.z += v[u][w].z; acc.w += v[u][w].w; }
  }
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) *out = acc.x;
}

template <int W, int U>
double gather_bw(const float4* buf, int rows, int ld4, int blocks, int threads, float* out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 2048;
  k_gather<W, U><<<blocks, threads>>>(buf, rows, ld4, 64, out);
  cudaEventRecord(a);
  k_gather<W, U><<<blocks, threads>>>(buf, rows, ld4, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return (double)blocks * (threads / 32) * iters * W * 512.0 / (ms / 1e3) / 1e9;
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
  // 2. gathers of W x 512-byte row chunks from a 20000-row slab of 1024 fp32 columns (82 MB)
  const int rows = 20000, ld4 = 256;
  double g512 = gather_bw<1, 8>(buf, rows, ld4, sms * 8, 256, out);
  double g1k = gather_bw<2, 8>(buf, rows, ld4, sms * 4, 256, out);
  double g2k = gather_bw<4, 4>(buf, rows, ld4, sms * 4, 256, out);
  double g4k = gather_bw<8, 2>(buf, rows, ld4, sms * 4, 256, out);
  double g1k_lo = gather_bw<2, 4>(buf, rows, ld4, sms * 8, 256, out);
  double l2_gather = g512;
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
         "\"l2_gather1k_gbs\": %.1f, \"l2_gather2k_gbs\": %.1f, \"l2_gather4k_gbs\": %.1f, \"l2_gather1k_u4_occ8_gbs\": %.1f, "
         "\"hbm_stream_read_gbs\": %.1f, \"err\": \"%s\"}\n",
         l2, sms, l2_stream, l2_gather, g1k, g2k, g4k, g1k_lo, hbm_read, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
