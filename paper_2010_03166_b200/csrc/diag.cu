// diag.cu -- machine-ceiling probe for the roofline of the aggregation kernels (SURVEY §8(d):
// "With X resident in L2, the real limit is L2->SM gather bandwidth ... Measure L2 read
// bandwidth on the box"). Not a step of the method: bench.py calls it in the same run as the
// step it reports, on the step's own activation buffer, so the SpMM's `roofline.peak` is a
// number measured beside it rather than read from an older file.
//
// The probe is the SpMM's gather stripped of the sparse structure: every warp gathers whole
// rows of X (row_floats fp32 columns, lane l loading bytes [32 l, 32 l + 32) with one 256-bit
// load, idle lanes re-reading the row's last 32 bytes exactly like k_spmm_wide), 8 rows in
// flight per warp, at rows drawn by a per-warp LCG (uniform over [0, rows)), accumulating with
// FFMA2-free plain adds; persistent grids of 2, 3 and 4 eight-warp CTAs per SM (the SpMM runs
// 2 or 3). Reported: gathered bytes / kernel time of the best grid.
#include <algorithm>

#include "common.cuh"

namespace gsg {
namespace {

__device__ __forceinline__ void ld256p(const void* p, float4 (&x)[2]) {
  asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(x[0].x), "=f"(x[0].y), "=f"(x[0].z), "=f"(x[0].w), "=f"(x[1].x), "=f"(x[1].y), "=f"(x[1].z),
                 "=f"(x[1].w)
               : "l"(p));
}

template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_gather_probe(const char* __restrict__ X, uint32_t rows,
                                                            uint64_t ld_bytes, uint32_t row_bytes, int iters,
                                                            float* __restrict__ sink) {
  constexpr int U = 8;
  const int lane = threadIdx.x & 31;
  const uint32_t lo = min(32u * lane, row_bytes - 32u);
  uint32_t s = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 2654435761u + 0x9E3779B9u;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int it = 0; it < iters; it += U) {
    float4 x[U][2];
#pragma unroll
    for (int u = 0; u < U; u++) {
      s = s * 1664525u + 1013904223u;
      const uint32_t r = (uint32_t)(((uint64_t)s * rows) >> 32);
      ld256p(X + (uint64_t)r * ld_bytes + lo, x[u]);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      acc.x += x[u][0].x + x[u][1].x;
      acc.y += x[u][0].y + x[u][1].y;
      acc.z += x[u][0].z + x[u][1].z;
      acc.w += x[u][0].w + x[u][1].w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 1.2345e-30f) *sink = acc.x;  // keeps the loads live
}

template <int MINB>
int probe_once(gsg_ctx* c, const float* X, int32_t rows, int64_t ldx, int32_t row_floats, float* sink,
               double* gbs) {
  const int grid = c->num_sms * MINB;
  const uint32_t row_bytes = (uint32_t)row_floats * 4u;
  // ~16 GB gathered per timed launch (~1 ms at the expected ceiling)
  int iters = (int)std::min<double>(1 << 20, 16e9 / ((double)grid * 8 * row_bytes));
  iters = std::max(64, iters / 8 * 8);
  const char* Xb = reinterpret_cast<const char*>(X);
  cudaEvent_t a = nullptr, b = nullptr;
  GSG_CUDA(cudaEventCreate(&a));
  GSG_CUDA(cudaEventCreate(&b));
  k_gather_probe<MINB><<<grid, 256, 0, c->stream>>>(Xb, (uint32_t)rows, (uint64_t)ldx * 4, row_bytes, 256, sink);
  cudaEventRecord(a, c->stream);
  k_gather_probe<MINB><<<grid, 256, 0, c->stream>>>(Xb, (uint32_t)rows, (uint64_t)ldx * 4, row_bytes, iters, sink);
  cudaEventRecord(b, c->stream);
  count_launch(c, 2);
  cudaError_t e = cudaEventSynchronize(b);
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (e != cudaSuccess) return cuda_fail(e, "gather probe");
  GSG_CUDA(cudaGetLastError());
  *gbs = (double)grid * 8 * iters * row_bytes / (ms / 1e3) / 1e9;
  return GSG_OK;
}

}  // namespace
}  // namespace gsg

using namespace gsg;

extern "C" GSG_API int gsg_diag_gather_ceiling(gsg_ctx_t c, const float* X, int32_t rows, int64_t ldx,
                                               int32_t row_floats, double* gbs) {
  GSG_CHECK(c && X && gbs, GSG_EINVAL, "NULL argument");
  GSG_CHECK(rows >= 1 && row_floats >= 8 && row_floats <= 256 && row_floats % 8 == 0 && ldx >= row_floats &&
                ldx % 8 == 0 && (uintptr_t)X % 32 == 0,
            GSG_EINVAL, "gather probe needs rows >= 1, row_floats in [8, 256] and a multiple of 8, ldx >= row_floats, "
                        "ldx %% 8 == 0 and a 32-byte aligned X (rows=%d row_floats=%d ldx=%lld)",
            rows, row_floats, (long long)ldx);
  DeviceGuard dg(c->device);
  DevBuf sink;
  if (int rc = sink.reserve(16)) return rc;
  double best = 0.0, g = 0.0;
  int rc = probe_once<2>(c, X, rows, ldx, row_floats, (float*)sink.ptr, &g);
  if (!rc) { best = std::max(best, g); rc = probe_once<3>(c, X, rows, ldx, row_floats, (float*)sink.ptr, &g); }
  if (!rc) { best = std::max(best, g); rc = probe_once<4>(c, X, rows, ldx, row_floats, (float*)sink.ptr, &g); }
  if (!rc) best = std::max(best, g);
  sink.release();
  if (rc) return rc;
  *gbs = best;
  return GSG_OK;
}
