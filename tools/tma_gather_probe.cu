// tma_gather_probe.cu -- measurement tool (not part of libgsg): is the SpMM's random-row gather
// limited by the bytes a warp can keep in flight in REGISTERS (the SpMM lands every gathered row
// in registers: ~192 rows per SM at 80 registers), or by the L2 itself?
// Two probes on the same L2-resident matrix (rows x 1024 fp32, random 1 KB chunk rows):
//   reg  : register landing, 8 rows in flight per warp (like gsg_diag_gather_ceiling)
//   tma  : cp.async.bulk (TMA) row copies into a per-warp shared-memory ring of R slots, each
//          completing on its own mbarrier; lanes then read their 32 bytes from smem and add.
//          In-flight rows per SM = CTAs x warps x R, bounded by shared memory, not registers.
// Prints one JSON line. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/tma_gather_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int R>
__global__ void __launch_bounds__(256) k_tma(const char* __restrict__ X, uint32_t rows, uint32_t ld_bytes,
                                              uint32_t row_bytes, int iters, float* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ring = sm + (size_t)warp * R * 1024;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)8 * R * 1024) + warp * R;
  uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 0x9E3779B9u;
  if (lane < R) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[lane])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  // lane j < R owns slot j: issues the copy of its slot's next row
  auto issue = [&](int j) {
    s = s * 1664525u + 1013904223u;
    const uint32_t r = (uint32_t)(((uint64_t)s * rows) >> 32);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[j])), "r"(row_bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(ring + j * 1024)),
        "l"(X + (uint64_t)r * ld_bytes), "r"(row_bytes), "r"(smem_u32(&bars[j]))
        : "memory");
  };
  if (lane < R) issue(lane);
  float4 acc0 = make_float4(0, 0, 0, 0), acc1 = acc0;
  uint32_t phase = 0;
  const uint32_t lo = min(32u * lane, row_bytes - 32u);
  for (int it = 0; it < iters; it += R) {
#pragma unroll 1
    for (int j = 0; j < R; j++) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
              smem_u32(&bars[j])),
          "r"(phase)
          : "memory");
      const float4 a = *reinterpret_cast<const float4*>(ring + j * 1024 + lo);
      const float4 b = *reinterpret_cast<const float4*>(ring + j * 1024 + lo + 16);
      acc0.x += a.x; acc0.y += a.y; acc0.z += a.z; acc0.w += a.w;
      acc1.x += b.x; acc1.y += b.y; acc1.z += b.z; acc1.w += b.w;
      __syncwarp();
      if (lane == j && it + R < iters) issue(j);  // refill the slot just read
    }
    phase ^= 1;
  }
  if (acc0.x + acc0.y + acc0.z + acc0.w + acc1.x + acc1.y + acc1.z + acc1.w == 1.2345e-30f) *sink = acc0.x;
}

__device__ __forceinline__ void ld256(const void* p, float4 (&x)[2]) {
  asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(x[0].x), "=f"(x[0].y), "=f"(x[0].z), "=f"(x[0].w), "=f"(x[1].x), "=f"(x[1].y), "=f"(x[1].z),
                 "=f"(x[1].w)
               : "l"(p));
}

template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_reg(const char* __restrict__ X, uint32_t rows, uint32_t ld_bytes,
                                                    uint32_t row_bytes, int iters, float* sink) {
  constexpr int U = 8;
  const int lane = threadIdx.x & 31;
  const uint32_t lo = min(32u * lane, row_bytes - 32u);
  uint32_t s = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 2654435761u + 0x9E3779B9u;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int it = 0; it < iters; it += U) {
    float4 x[U][2];
#pragma unroll
    for (int u = 0; u < U; u++) {
      s = s * 1664525u + 1013904223u;
      ld256(X + (uint64_t)(uint32_t)(((uint64_t)s * rows) >> 32) * ld_bytes + lo, x[u]);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      acc.x += x[u][0].x + x[u][1].x; acc.y += x[u][0].y + x[u][1].y;
      acc.z += x[u][0].z + x[u][1].z; acc.w += x[u][0].w + x[u][1].w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 1.2345e-30f) *sink = acc.x;
}

// tile::gather4 TMA: ONE instruction brings 4 random 1 KB rows (box {256 floats, 1 row}, four
// row coordinates) into a 4 KB shared-memory slot; per warp R slots, each on its own mbarrier.
// Lane 0 issues; after a slot's wait every lane reads its 32 bytes of each of the 4 rows.
template <int R>
__global__ void __launch_bounds__(256) k_g4(const __grid_constant__ CUtensorMap tm, uint32_t rows, int iters,
                                             uint32_t row_bytes, float* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ring = sm + (size_t)warp * R * 4096;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)8 * R * 4096) + warp * R;
  uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 0x9E3779B9u;
  if (lane < R) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[lane])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](int j) {  // lane 0 only
    int r[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      s = s * 1664525u + 1013904223u;
      r[q] = (int)(((uint64_t)s * rows) >> 32);
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[j])), "r"(4 * row_bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        ::"r"(smem_u32(ring + j * 4096)), "l"(&tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]),
        "r"(smem_u32(&bars[j]))
        : "memory");
  };
  if (lane == 0)
    for (int j = 0; j < R; j++) issue(j);
  float4 acc0 = make_float4(0, 0, 0, 0), acc1 = acc0;
  uint32_t phase = 0;
  const uint32_t lo = min(32u * lane, row_bytes - 32u);
  for (int it = 0; it < iters; it += 4 * R) {
#pragma unroll 1
    for (int j = 0; j < R; j++) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
              smem_u32(&bars[j])),
          "r"(phase)
          : "memory");
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const float4 a = *reinterpret_cast<const float4*>(ring + j * 4096 + q * row_bytes + lo);
        const float4 b = *reinterpret_cast<const float4*>(ring + j * 4096 + q * row_bytes + lo + 16);
        acc0.x += a.x; acc0.y += a.y; acc0.z += a.z; acc0.w += a.w;
        acc1.x += b.x; acc1.y += b.y; acc1.z += b.z; acc1.w += b.w;
      }
      __syncwarp();
      if (lane == 0 && it + 4 * R < iters) issue(j);  // refill the slot just read
    }
    phase ^= 1;
  }
  if (acc0.x + acc0.y + acc0.z + acc0.w + acc1.x + acc1.y + acc1.z + acc1.w == 1.2345e-30f) *sink = acc0.x;
}

template <typename F>
double timeit(F launch, double bytes) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch(64);
  cudaEventRecord(a);
  launch(-1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return bytes / (ms / 1e3) / 1e9;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t rows = 20000, ldb = 4096;
  char* X;
  cudaMalloc(&X, (size_t)rows * ldb);
  cudaMemset(X, 0, (size_t)rows * ldb);
  float* sink;
  cudaMalloc(&sink, 16);
  printf("{");
  for (uint32_t rb : {1024u, 800u}) {
    const int iters = 4096;
    double best_reg = 0;
    int best_reg_cfg = 0;
    auto reg = [&](auto kern, int minb) {
      const int grid = sms * minb;
      double g = timeit([&](int it) { kern<<<grid, 256>>>(X, rows, ldb, rb, it < 0 ? iters : it, sink); },
                        (double)grid * 8 * iters * rb);
      if (g > best_reg) { best_reg = g; best_reg_cfg = minb; }
    };
    reg(k_reg<2>, 2);
    reg(k_reg<3>, 3);
    reg(k_reg<4>, 4);
    printf("\"reg_%u_gbs\": %.1f, \"reg_%u_ctas\": %d, ", rb, best_reg, rb, best_reg_cfg);
    auto tma = [&](auto kern, int R, int ctas) {
      const size_t smem = (size_t)8 * R * 1024 + 8 * R * 8;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int grid = sms * ctas;
      double g = timeit([&](int it) { kern<<<grid, 256, smem>>>(X, rows, ldb, rb, it < 0 ? iters : it, sink); },
                        (double)grid * 8 * iters * rb);
      printf("\"tma_%u_R%d_c%d_gbs\": %.1f, ", rb, R, ctas, g);
    };
    tma(k_tma<8>, 8, 1);
    tma(k_tma<8>, 8, 2);
    tma(k_tma<8>, 8, 3);
    tma(k_tma<16>, 16, 1);
    tma(k_tma<24>, 24, 1);
  }
  {  // gather4 TMA probe on the same matrix (fp32 view: rows x ldb/4, box 256 x 1)
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    CUtensorMap tm;
    cuuint64_t gdim[2] = {ldb / 4, rows};
    cuuint64_t gstr[1] = {ldb};
    cuuint32_t box[2] = {256, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("\"g4_encode\": %d, ", (int)cr);
    auto g4 = [&](auto kern, int R, int ctas) {
      const size_t smem = (size_t)8 * R * 4096 + 8 * R * 8;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int grid = sms * ctas;
      const int iters = 4096;
      double g = timeit([&](int it) { kern<<<grid, 256, smem>>>(tm, rows, it < 0 ? iters : it, 1024u, sink); },
                        (double)grid * 8 * iters * 1024);
      printf("\"g4_1024_R%d_c%d_gbs\": %.1f, \"g4_err_R%d_c%d\": \"%s\", ", R, ctas, g, R, ctas,
             cudaGetErrorString(cudaGetLastError()));
    };
    g4(k_g4<1>, 1, 1);
    g4(k_g4<2>, 2, 1);
    g4(k_g4<3>, 3, 1);
    g4(k_g4<6>, 6, 1);
    g4(k_g4<2>, 2, 2);
    g4(k_g4<3>, 3, 2);
  }
  printf("\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
