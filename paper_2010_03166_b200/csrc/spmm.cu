// spmm.cu -- SURVEY §8(a) rows a2 (P = Â X) and a7 (dX = Âᵀ T [⊙ 1[H_below > 0]]).
//
// The product is Alg. 6's feature propagation re-designed for sm_100a:
//   * The paper splits the feature columns into Q_f slabs, one per core, so each core's slab
//     fits its private cache (Theorem 2). On B200 every SM should instead work on
//     the SAME column slab at a time so the slab is shared through the 126 MB L2: tasks are
//     ordered chunk-major (all rows of column chunk 0, then chunk 1, ...), so the concurrently
//     running warps touch one n x 128-column slab (10 MB at n = 20,000).
//   * One lane owns one float4 column group; a warp task is one (row, <=128-column chunk)
//     pair; neighbor (idx, val) pairs are loaded 32 at a time and broadcast with __shfl_sync;
//     8 independent 16-byte row gathers are in flight per lane.
//   * Degree bins (built by normalize): rows are visited in descending degree order, and
//     "heavy" rows (deg' >= 256) are split across the 8 warps of a CTA whose partial sums are
//     reduced through shared memory in a fixed warp order.
//   * Narrow features (f <= 64) use sub-warp groups of 4/8/16 lanes, one row per group.
//   * Persistent grid (SMs x resident CTAs) with a static round-robin task schedule read
//     from device counters, so the launch needs no host synchronization.
// Every output row is accumulated in a fixed order -> bitwise reproducible.
#include <cuda_bf16.h>

#include "common.cuh"

namespace gsg {
namespace {

struct SpmmArgs {
  int n, f4, nchunks, cw;
  const int32_t* __restrict__ rowptr;
  const int32_t* __restrict__ col;
  const float* __restrict__ val;
  const float4* __restrict__ X;
  int64_t ldx4;
  float4* __restrict__ Y;
  int64_t ldy4;
  uint2* __restrict__ Ylp;   // 4 bf16 per uint2
  int64_t ldylp4;
  const float4* __restrict__ mask;
  int64_t ldm4;
  const int32_t* __restrict__ perm;
  const int32_t* __restrict__ n_heavy_ptr;
};

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

__device__ __forceinline__ void fma4(float a, const float4& v, float4& acc) {
  acc.x = fmaf(a, v.x, acc.x);
  acc.y = fmaf(a, v.y, acc.y);
  acc.z = fmaf(a, v.z, acc.z);
  acc.w = fmaf(a, v.w, acc.w);
}

__device__ __forceinline__ float4 ldx(const float4* p) { return __ldg(p); }

// Full-warp accumulation of sum_{k in [b, e)} val[k] * X[col[k], c4] (c4 = this lane's float4).
__device__ __forceinline__ float4 warp_row_sum(const SpmmArgs& a, int b, int e, int c4, bool act, int lane) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* Xc = a.X + c4;
  for (int k0 = b; k0 < e; k0 += 32) {
    const int k = k0 + lane;
    const int cnt = min(32, e - k0);
    const int cj = k < e ? __ldg(a.col + k) : 0;
    const float aj = k < e ? __ldg(a.val + k) : 0.f;
    int j = 0;
    for (; j + 8 <= cnt; j += 8) {
      int c[8];
      float w[8];
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        c[u] = __shfl_sync(0xffffffffu, cj, j + u);
        w[u] = __shfl_sync(0xffffffffu, aj, j + u);
      }
      if (act) {
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] = ldx(Xc + (int64_t)c[u] * a.ldx4);
#pragma unroll
        for (int u = 0; u < 8; u++) fma4(w[u], v[u], acc);
      }
    }
    for (; j < cnt; j++) {
      const int c = __shfl_sync(0xffffffffu, cj, j);
      const float w = __shfl_sync(0xffffffffu, aj, j);
      if (act) fma4(w, ldx(Xc + (int64_t)c * a.ldx4), acc);
    }
  }
  return acc;
}

// Sub-warp (group of G lanes, one row) accumulation; no shuffles (groups diverge).
__device__ __forceinline__ float4 group_row_sum(const SpmmArgs& a, int b, int e, int c4, bool act) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* Xc = a.X + c4;
  int k = b;
  for (; k + 4 <= e; k += 4) {
    int c[4];
    float w[4];
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; u++) { c[u] = __ldg(a.col + k + u); w[u] = __ldg(a.val + k + u); }
    if (act) {
#pragma unroll
      for (int u = 0; u < 4; u++) v[u] = ldx(Xc + (int64_t)c[u] * a.ldx4);
#pragma unroll
      for (int u = 0; u < 4; u++) fma4(w[u], v[u], acc);
    }
  }
  for (; k < e; k++) {
    const int c = __ldg(a.col + k);
    const float w = __ldg(a.val + k);
    if (act) fma4(w, ldx(Xc + (int64_t)c * a.ldx4), acc);
  }
  return acc;
}

__device__ __forceinline__ void store_row(const SpmmArgs& a, int row, int c4, float4 acc) {
  if (a.mask) {
    const float4 m = __ldg(a.mask + (int64_t)row * a.ldm4 + c4);
    acc.x = m.x > 0.f ? acc.x : 0.f;
    acc.y = m.y > 0.f ? acc.y : 0.f;
    acc.z = m.z > 0.f ? acc.z : 0.f;
    acc.w = m.w > 0.f ? acc.w : 0.f;
  }
  a.Y[(int64_t)row * a.ldy4 + c4] = acc;
  if (a.Ylp) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y);
    __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z, acc.w);
    uint2 p;
    p.x = *reinterpret_cast<uint32_t*>(&lo);
    p.y = *reinterpret_cast<uint32_t*>(&hi);
    a.Ylp[(int64_t)row * a.ldylp4 + c4] = p;
  }
}

template <int G>
__global__ void __launch_bounds__(kThreads) k_spmm(SpmmArgs a) {
  __shared__ float4 part[kWarps][32];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int n_heavy = *a.n_heavy_ptr;
  const int n_light = a.n - n_heavy;

  // ---- phase 1: heavy rows, one CTA per (row, chunk), neighbors split across 8 warps ----
  const int64_t H = (int64_t)n_heavy * a.nchunks;
  for (int64_t t = blockIdx.x; t < H; t += gridDim.x) {
    const int chunk = (int)(t / n_heavy);
    const int row = a.perm[t % n_heavy];
    const int b = a.rowptr[row], e = a.rowptr[row + 1];
    const int seg = (e - b + kWarps - 1) / kWarps;
    const int w0 = min(e, b + warp * seg), w1 = min(e, w0 + seg);
    const int c4 = chunk * a.cw + lane;
    const bool act = lane < a.cw && c4 < a.f4;
    part[warp][lane] = warp_row_sum(a, w0, w1, c4, act, lane);
    __syncthreads();
    if (warp == 0) {
      float4 s = part[0][lane];
#pragma unroll
      for (int w = 1; w < kWarps; w++) {
        const float4 p = part[w][lane];
        s.x += p.x; s.y += p.y; s.z += p.z; s.w += p.w;
      }
      if (act) store_row(a, row, c4, s);
    }
    __syncthreads();
  }

  // ---- phase 2: light rows ----
  if (G == 32) {
    const int64_t L = (int64_t)n_light * a.nchunks;
    const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
    const int64_t GW = (int64_t)gridDim.x * kWarps;
    for (int64_t t = gw; t < L; t += GW) {
      const int chunk = (int)(t / n_light);
      const int row = a.perm[n_heavy + (int)(t % n_light)];
      const int c4 = chunk * a.cw + lane;
      const bool act = lane < a.cw && c4 < a.f4;
      const float4 acc = warp_row_sum(a, a.rowptr[row], a.rowptr[row + 1], c4, act, lane);
      if (act) store_row(a, row, c4, acc);
    }
  } else {
    constexpr int PER = 32 / G;
    const int g = lane / G, gl = lane % G;
    const int64_t gid = ((int64_t)blockIdx.x * kWarps + warp) * PER + g;
    const int64_t GN = (int64_t)gridDim.x * kWarps * PER;
    const bool act = gl < a.f4;
    for (int64_t t = gid; t < n_light; t += GN) {
      const int row = a.perm[n_heavy + (int)t];
      const float4 acc = group_row_sum(a, a.rowptr[row], a.rowptr[row + 1], gl, act);
      if (act) store_row(a, row, gl, acc);
    }
  }
}

template <int G>
int launch_g(gsg_ctx* ctx, const SpmmArgs& a, int64_t tasks) {
  static int occ = -1;
  if (occ < 0) {
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_spmm<G>, kThreads, 0) != cudaSuccess || o < 1) o = 1;
    occ = o;
  }
  int64_t want = (tasks + kWarps - 1) / kWarps;
  int64_t grid = (int64_t)ctx->num_sms * occ;
  if (want < grid) grid = want;
  if (grid < 1) grid = 1;
  k_spmm<G><<<(int)grid, kThreads, 0, ctx->stream>>>(a);
  count_launch(ctx);
  GSG_CUDA(cudaGetLastError());
  return GSG_OK;
}

}  // namespace

int spmm_launch(gsg_ctx* ctx, const gsg_subgraph* sg, int transpose, int f, const float* X, int64_t ldx,
                float* Y, int64_t ldy, void* Ylp, int64_t ldylp, const float* mask, int64_t ldm) {
  GSG_CHECK(sg->norm_mode >= 0, GSG_EINVAL, "subgraph not normalized (call gsg_subgraph_normalize)");
  GSG_CHECK(f >= 1, GSG_EINVAL, "f must be >= 1 (got %d)", f);
  GSG_CHECK(X && Y, GSG_EINVAL, "X and Y must be non-NULL");
  GSG_CHECK(ldx >= f && ldx % 4 == 0, GSG_EINVAL, "ldx=%lld must be >= f=%d and a multiple of 4", (long long)ldx, f);
  GSG_CHECK(ldy >= f && ldy % 4 == 0, GSG_EINVAL, "ldy=%lld must be >= f=%d and a multiple of 4", (long long)ldy, f);
  GSG_CHECK(((uintptr_t)X | (uintptr_t)Y) % 16 == 0, GSG_EINVAL, "X/Y must be 16-byte aligned");
  GSG_CHECK(!Ylp || (ldylp >= f && ldylp % 8 == 0 && (uintptr_t)Ylp % 16 == 0), GSG_EINVAL,
            "bf16 output needs ldylp >= f, ldylp %% 8 == 0 and 16-byte alignment");
  GSG_CHECK(!mask || (ldm >= f && ldm % 4 == 0 && (uintptr_t)mask % 16 == 0), GSG_EINVAL,
            "mask needs ldm >= f, ldm %% 4 == 0 and 16-byte alignment");
  GSG_CHECK(X != Y, GSG_EINVAL, "Y must not alias X");
  if (sg->n == 0) return GSG_OK;
  // algorithmic (effective gather) bytes, SURVEY §8(d)
  const double nh = (double)sg->nnz_hat, nn = (double)sg->n;
  ProfScope ps(ctx, GSG_K_SPMM, 4.0 * nh * f + 8.0 * nh + 4.0 * (nn + 1) + 4.0 * nn * f, 2.0 * nh * f);
  SpmmArgs a;
  a.n = sg->n;
  a.f4 = (f + 3) / 4;
  a.rowptr = sg->rowptr;
  a.col = sg->col;
  a.val = transpose ? sg->valT : sg->val;
  a.X = reinterpret_cast<const float4*>(X);
  a.ldx4 = ldx / 4;
  a.Y = reinterpret_cast<float4*>(Y);
  a.ldy4 = ldy / 4;
  a.Ylp = reinterpret_cast<uint2*>(Ylp);
  a.ldylp4 = ldylp / 4;
  a.mask = reinterpret_cast<const float4*>(mask);
  a.ldm4 = ldm / 4;
  a.perm = sg->perm;
  a.n_heavy_ptr = sg->counters + kBins;
  if (a.f4 > 16) {
    a.nchunks = (a.f4 + 31) / 32;
    a.cw = (a.f4 + a.nchunks - 1) / a.nchunks;
    return launch_g<32>(ctx, a, (int64_t)sg->n * a.nchunks);
  }
  a.nchunks = 1;
  a.cw = a.f4;
  if (a.f4 > 8) return launch_g<16>(ctx, a, (int64_t)sg->n / 2 + 1);
  if (a.f4 > 4) return launch_g<8>(ctx, a, (int64_t)sg->n / 4 + 1);
  return launch_g<4>(ctx, a, (int64_t)sg->n / 8 + 1);
}

}  // namespace gsg
