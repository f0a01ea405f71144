// spmm.cu -- SURVEY §8(a) rows a2 (P = Â X) and a7 (dX = Âᵀ T [⊙ 1[H_below > 0]]).
//
// The product is Alg. 6's feature propagation re-designed for sm_100a:
//   * The paper splits the feature columns into Q_f slabs, one per core, so each core's slab
//     fits its private cache (Theorem 2). On B200 every SM instead works on the
//     SAME column slab at a time so the slab is shared through the 126 MB L2: tasks are
//     ordered chunk-major (all rows of column chunk 0, then chunk 1, ...), so the concurrently
//     running warps touch one n x 256-column slab (20 MB at n = 20,000).
//   * A warp task is one (row, <= 256-column chunk) pair; lane l owns the float4 column pair
//     2l, 2l + 1 of the chunk, so every neighbor costs one 32-bit offset broadcast and ONE
//     coalesced 1 KB row gather (LDG.E.256) -- when X is 32-byte aligned with ldx % 8 == 0;
//     otherwise lane l owns float4 columns l and l + 32 and gathers with two LDG.128.
//     Neighbor (offset, value) pairs are staged 32 at a time in shared memory and read back as
//     128-bit broadcasts (two pairs per LDS.128); 8 neighbors' gathers (8 KB per warp) are in
//     flight per iteration; accumulation uses packed
//     fp32x2 FMAs (FFMA2). The kernel is bound by L2->SM gather throughput (X is L2-resident),
//     so instructions per gathered byte are what the design minimizes.
//   * Degree bins (built by normalize): rows are visited in descending degree order, and
//     "heavy" rows (deg' >= 256) are split across the 8 warps of a CTA whose partial sums are
//     reduced through shared memory in a fixed warp order.
//   * Narrow features (f <= 64) use sub-warp groups of 4/8/16 lanes, one row per group.
//   * Persistent grid (SMs x resident CTAs) with a static round-robin task schedule read
//     from device counters, so the launch needs no host synchronization.
// Every output row is accumulated in a fixed order -> bitwise reproducible.
#include <cuda_bf16.h>

#include <algorithm>

#include <cstdlib>

#include <atomic>
#include <type_traits>

#include "common.cuh"

namespace gsg {
namespace {

struct SpmmArgs {
  int n, f4, nchunks, cw;
  const int32_t* __restrict__ rowptr;
  const int32_t* __restrict__ col;
  const float* __restrict__ val;
  const float4* __restrict__ X;
  uint32_t ldx4;             // row stride of X in float4
  uint32_t ldx16;            // row stride of X in bytes (n * ldx * 4 < 2^32 checked on the host)
  float4* __restrict__ Y;
  int64_t ldy4;
  uint2* __restrict__ Ylp;   // 4 bf16 per uint2
  int64_t ldylp4;
  const float4* __restrict__ mask;
  int relu;                  // epilogue ReLU (chain order 2 forward: H = ReLU(Â (X W)))
  int accum;                 // epilogue Y = Y + result, before the gate (GraphSAGE dX = self + neighbor terms)
  int64_t ldm4;
  const int32_t* __restrict__ perm;
  const int32_t* __restrict__ n_heavy_ptr;
  const int32_t* __restrict__ bucket_counts;  // [kBins] rows per log2 degree bucket
  const int32_t* __restrict__ n_mega_ptr;
  float4* __restrict__ mega_ws;   // [mega row][segment][f4] partials (cap_mega rows)
  int* __restrict__ mega_ctr;     // [mega row][chunk] arrival counters (zero between launches)
  int cap_mega;                   // mega rows the workspace holds (more are processed whole)
  const uint32_t* __restrict__ mbits;  // ReLU' gate as a bitmask (gsg.h), replaces mask
  int64_t ldmb;
  uint32_t* __restrict__ obits;        // relu: also OR 1[Y > 0] into this bitmask (zeroed first)
  int64_t ldob;
  int f;
  int w256;                  // 1: lanes gather 32-byte column pairs with 256-bit loads (X 32-B aligned, ldx % 8 == 0)
  int heavy_bucket;          // rows of degree bucket >= this are CTA-split ("heavy"; the first of perm)
  int seg_align;             // CTA-split rows: each warp's share rounded up to a multiple of this
  int hseg;                  // 1: heavy rows as warp segments (htask) instead of CTA-split rows
  const int4* __restrict__ htask;      // heavy-row segments (normalize): row, k_begin, k_end, first
  const int32_t* __restrict__ hcount;  // segments of the row whose first segment is the index
  const int32_t* __restrict__ n_hseg_ptr;
  float4* __restrict__ hseg_ws;        // [segment][f4] partial sums of multi-segment rows
  int* __restrict__ hseg_ctr;          // [first segment][chunk] arrival counters (zero between launches)
  int* __restrict__ task_ctr;          // dyn: [0] warp tasks handed out past the first GW, [1] CTAs done (zero between launches)
  int dyn;                             // 1: warp tasks past the first round are claimed from task_ctr
  int tailg;                           // > 0: the last column chunk (<= 2*tailg float4) is gathered by
                                       // lane groups of tailg, 32/tailg neighbors per warp instruction
};

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int V = 2;   // float4 per lane per neighbor (full-warp path)
constexpr int U = 8;   // neighbors per unrolled iteration
constexpr int kRing = 1;  // heavy-row tasks whose partial sums a CTA holds at once

// acc += a * x on packed fp32 pairs (FFMA2, round-to-nearest per element: identical to two FFMAs)
__device__ __forceinline__ void fma2(float2& acc, float a, float2 x) {
  unsigned long long r;
  const unsigned long long aa = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
  const unsigned long long xx = ((unsigned long long)__float_as_uint(x.y) << 32) | __float_as_uint(x.x);
  const unsigned long long cc = ((unsigned long long)__float_as_uint(acc.y) << 32) | __float_as_uint(acc.x);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(aa), "l"(xx), "l"(cc));
  acc.x = __uint_as_float((uint32_t)r);
  acc.y = __uint_as_float((uint32_t)(r >> 32));
}

struct Acc {
  float2 v[2 * V];
};

__device__ __forceinline__ void acc_fma(Acc& A, float w, const float4 (&x)[V]) {
#pragma unroll
  for (int q = 0; q < V; q++) {
    fma2(A.v[2 * q], w, make_float2(x[q].x, x[q].y));
    fma2(A.v[2 * q + 1], w, make_float2(x[q].z, x[q].w));
  }
}

__device__ __forceinline__ const float4* row_ptr(const float4* X, uint32_t byte_off) {
  return reinterpret_cast<const float4*>(reinterpret_cast<const char*>(X) + byte_off);
}

// Full-warp accumulation over neighbors [b, e) of this lane's float4 columns. Lanes whose
// column falls outside the chunk read the chunk's last column instead (same sectors as an
// active lane: no extra traffic, no predication); their sums are never stored.
// FULL: every lane's columns are inside the chunk, so the second gather is the first + 512 B
// (an immediate offset): per neighbor one 64-bit address add, two LDG.128, four FFMA2.
template <bool FULL>
__device__ __forceinline__ void warp_row_sum(const SpmmArgs& a, int2* __restrict__ st, int b, int e,
                                             uint32_t lo0, uint32_t lo1, int lane, Acc& A) {
  const float4* X = a.X;
  const float4* X0 = row_ptr(X, lo0);
#pragma unroll
  for (int q = 0; q < 2 * V; q++) A.v[q] = make_float2(0.f, 0.f);
  for (int k0 = b; k0 < e; k0 += 32) {
    const int k = k0 + lane;
    if (k < e) st[lane] = make_int2((int)((uint32_t)__ldg(a.col + k) * a.ldx16), __float_as_int(__ldg(a.val + k)));
    __syncwarp();
    const int cnt = min(32, e - k0);
    int j = 0;
    for (; j + U <= cnt; j += U) {
      int4 p[U / 2];
#pragma unroll
      for (int q = 0; q < U / 2; q++) p[q] = reinterpret_cast<const int4*>(st)[(j >> 1) + q];
      float4 x[U][V];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const uint32_t off = (u & 1) ? (uint32_t)p[u >> 1].z : (uint32_t)p[u >> 1].x;
        if (FULL) {
          const float4* r = row_ptr(X0, off);
          x[u][0] = __ldg(r);
          if (V == 2) x[u][1] = __ldg(r + 32);
        } else {
          x[u][0] = __ldg(row_ptr(X, off + lo0));
          if (V == 2) x[u][1] = __ldg(row_ptr(X, off + lo1));
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const float w = __int_as_float((u & 1) ? p[u >> 1].w : p[u >> 1].y);
        acc_fma(A, w, x[u]);
      }
    }
    for (; j < cnt; j++) {
      const int2 p = st[j];
      float4 x[V];
      x[0] = __ldg(row_ptr(X, (uint32_t)p.x + lo0));
      if (V == 2) x[1] = __ldg(row_ptr(X, (uint32_t)p.x + lo1));
      acc_fma(A, __int_as_float(p.y), x);
    }
    __syncwarp();
  }
}

// One 256-bit gather (LDG.E.256): the lane's two adjacent float4 columns of one X row.
__device__ __forceinline__ void ld256(const void* p, float4 (&x)[2]) {
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(x[0].x), "=f"(x[0].y), "=f"(x[0].z), "=f"(x[0].w), "=f"(x[1].x), "=f"(x[1].y), "=f"(x[1].z),
        "=f"(x[1].w)
      : "l"(p));
}

// warp_row_sum with 256-bit gathers: lane l owns float4 columns 2l and 2l + 1 of the chunk
// (lo = byte offset of that pair; idle lanes re-read the chunk's last pair), so a 1 KB chunk
// row is ONE warp-wide load instruction instead of two 512-byte ones -- half the load
// instructions and L1 requests per gathered byte, same bytes and registers in flight.
template <int UU>
__device__ __forceinline__ void warp_row_sum256(const SpmmArgs& a, int2* __restrict__ st, int b, int e, uint32_t lo,
                                                int lane, Acc& A) {
  static_assert(UU % 2 == 0 && UU <= 8, "UU: even, <= 8");
  const char* X0 = reinterpret_cast<const char*>(a.X) + lo;
#pragma unroll
  for (int q = 0; q < 2 * V; q++) A.v[q] = make_float2(0.f, 0.f);
  for (int k0 = b; k0 < e; k0 += 32) {
    const int k = k0 + lane;
    int2 pr = make_int2(0, 0);
    if (k < e) pr = make_int2((int)((uint32_t)__ldg(a.col + k) * a.ldx16), __float_as_int(__ldg(a.val + k)));
    // slots past the row's end gather the group's first neighbor row again with weight 0, so the
    // last (partial) batch is an ordinary U-wide batch: one round trip instead of one per
    // remaining neighbor, and no predication (which made ptxas spread the gathers out)
    const int off0 = __shfl_sync(0xffffffffu, pr.x, 0);
    if (k >= e) pr = make_int2(off0, 0);
    st[lane] = pr;
    if (UU % 8 != 0 && lane < 8) st[32 + lane] = make_int2(off0, 0);  // a batch may run past slot 31
    __syncwarp();
    const int cnt = min(32, e - k0);
    for (int j = 0; j < cnt; j += UU) {
      int4 p[UU / 2];
#pragma unroll
      for (int q = 0; q < UU / 2; q++) p[q] = reinterpret_cast<const int4*>(st)[(j >> 1) + q];
      float4 x[UU][V];
#pragma unroll
      for (int u = 0; u < UU; u++) ld256(X0 + ((u & 1) ? (uint32_t)p[u >> 1].z : (uint32_t)p[u >> 1].x), x[u]);
#pragma unroll
      for (int u = 0; u < UU; u++) acc_fma(A, __int_as_float((u & 1) ? p[u >> 1].w : p[u >> 1].y), x[u]);
    }
    __syncwarp();
  }
}

// The last, narrow column chunk of a row (r <= 2G float4, e.g. f = 300: 64 + 11 float4) with lane
// groups of G: group g gathers neighbors g, g + 32/G, ... of the staged 32, so one warp-wide 256-bit
// load instruction moves 32/G neighbor rows instead of one row with 32 - r/2 idle lanes (f = 300:
// 1.25 instead of 2 load instructions per neighbor). Batches of 8 / 4 / 2 / 1 instructions cover
// only the staged neighbors. The group sums are combined in a fixed tree (g0 + g1) + (g2 + g3) into
// lanes 0..G-1 (every other lane's columns lie past the chunk and are never stored): deterministic.
template <int G>
__device__ __forceinline__ void warp_row_sum256_grp(const SpmmArgs& a, int2* __restrict__ st, int b, int e, uint32_t lo,
                                                    int lane, Acc& A) {
  constexpr int NG = 32 / G;
  const int g = lane / G;
  const char* X0 = reinterpret_cast<const char*>(a.X) + lo;
#pragma unroll
  for (int q = 0; q < 2 * V; q++) A.v[q] = make_float2(0.f, 0.f);
  auto batch = [&](auto ub, int i) {
    constexpr int UB = decltype(ub)::value;
    int2 p[UB];
#pragma unroll
    for (int u = 0; u < UB; u++) p[u] = st[(i + u) * NG + g];
    float4 x[UB][V];
#pragma unroll
    for (int u = 0; u < UB; u++) ld256(X0 + (uint32_t)p[u].x, x[u]);
#pragma unroll
    for (int u = 0; u < UB; u++) acc_fma(A, __int_as_float(p[u].y), x[u]);
  };
  for (int k0 = b; k0 < e; k0 += 32) {
    const int k = k0 + lane;
    int2 pr = make_int2(0, 0);
    if (k < e) pr = make_int2((int)((uint32_t)__ldg(a.col + k) * a.ldx16), __float_as_int(__ldg(a.val + k)));
    const int off0 = __shfl_sync(0xffffffffu, pr.x, 0);
    if (k >= e) pr = make_int2(off0, 0);  // padding slots: the first neighbor's row again, weight 0
    st[lane] = pr;
    __syncwarp();
    const int ni = (min(32, e - k0) + NG - 1) / NG;  // warp instructions for the staged neighbors
    int i = 0;
    for (; i + 8 <= ni; i += 8) batch(std::integral_constant<int, 8>{}, i);
    if (i + 4 <= ni) { batch(std::integral_constant<int, 4>{}, i); i += 4; }
    if (i + 2 <= ni) { batch(std::integral_constant<int, 2>{}, i); i += 2; }
    if (i < ni) batch(std::integral_constant<int, 1>{}, i);
    __syncwarp();
  }
#pragma unroll
  for (int sh = G; sh < 32; sh <<= 1) {
#pragma unroll
    for (int q = 0; q < 2 * V; q++) {
      A.v[q].x += __shfl_down_sync(0xffffffffu, A.v[q].x, sh);
      A.v[q].y += __shfl_down_sync(0xffffffffu, A.v[q].y, sh);
    }
  }
}

// W256 gather of one (row range, chunk) task: the grouped tail path for the last chunk when
// a.tailg is set, else one row per warp instruction
template <int UU>
__device__ __forceinline__ void gather256(const SpmmArgs& a, int2* __restrict__ st, int b, int e, int chunk, int c0,
                                          int lim, int lane, Acc& A) {
  if (a.tailg && chunk == a.nchunks - 1) {
    const int G = a.tailg;
    const uint32_t lo = 16u * (c0 + min(2 * (lane & (G - 1)), (lim - c0 - 1) & ~1));
    if (G == 8) warp_row_sum256_grp<8>(a, st, b, e, lo, lane, A);
    else warp_row_sum256_grp<16>(a, st, b, e, lo, lane, A);
    return;
  }
  warp_row_sum256<UU>(a, st, b, e, 16u * (c0 + min(2 * lane, (lim - c0 - 1) & ~1)), lane, A);
}

// Sub-warp (group of G lanes, one row) accumulation; no shuffles (groups diverge).
__device__ __forceinline__ void fma4(float4& acc, float w, const float4& v) {
  acc.x = fmaf(w, v.x, acc.x);
  acc.y = fmaf(w, v.y, acc.y);
  acc.z = fmaf(w, v.z, acc.z);
  acc.w = fmaf(w, v.w, acc.w);
}

// 8 neighbors per batch: the 8 (col, val) loads, then the 8 row gathers, are independent, so a
// row costs one dependent round trip per 8 neighbors; the last batch is predicated.
__device__ __forceinline__ float4 group_row_sum(const SpmmArgs& a, int b, int e, int c4, bool act) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* Xc = a.X + c4;
  for (int k = b; k < e; k += 8) {
    uint32_t c[8];
    float w[8];
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const bool ok = k + u < e;
      c[u] = ok ? (uint32_t)__ldg(a.col + k + u) * a.ldx4 : 0u;
      w[u] = ok ? __ldg(a.val + k + u) : 0.f;
    }
    if (act) {
#pragma unroll
      for (int u = 0; u < 8; u++) v[u] = k + u < e ? __ldg(Xc + c[u]) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (k + u < e) fma4(acc, w[u], v[u]);
    }
  }
  return acc;
}

// mw: the gate word of (row, c4) already loaded by the caller (bitmask gate), else nullptr
__device__ __forceinline__ void store_row(const SpmmArgs& a, int row, int c4, float4 acc,
                                          const uint32_t* mw = nullptr) {
  if (a.accum) {
    const float4 o = a.Y[(int64_t)row * a.ldy4 + c4];
    acc.x += o.x; acc.y += o.y; acc.z += o.z; acc.w += o.w;
  }
  if (a.relu) {
    acc.x = fmaxf(acc.x, 0.f);
    acc.y = fmaxf(acc.y, 0.f);
    acc.z = fmaxf(acc.z, 0.f);
    acc.w = fmaxf(acc.w, 0.f);
    if (a.obits) {
      // this lane's 4 columns are one nibble of a 32-column word; 8 lanes share a word
      uint32_t nib = (acc.x > 0.f ? 1u : 0u) | (acc.y > 0.f ? 2u : 0u) | (acc.z > 0.f ? 4u : 0u) | (acc.w > 0.f ? 8u : 0u);
      const int valid = a.f - 4 * c4;
      if (valid < 4) nib &= (1u << valid) - 1u;
      if (nib) atomicOr(a.obits + (int64_t)row * a.ldob + (c4 >> 3), nib << ((c4 & 7) * 4));
    }
  }
  if (a.mbits) {
    const uint32_t m = (mw ? *mw : __ldg(a.mbits + (int64_t)row * a.ldmb + (c4 >> 3))) >> ((c4 & 7) * 4);
    acc.x = m & 1u ? acc.x : 0.f;
    acc.y = m & 2u ? acc.y : 0.f;
    acc.z = m & 4u ? acc.z : 0.f;
    acc.w = m & 8u ? acc.w : 0.f;
  } else if (a.mask) {
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

__device__ __forceinline__ float4 acc_part(const Acc& A, int q) {
  return make_float4(A.v[2 * q].x, A.v[2 * q].y, A.v[2 * q + 1].x, A.v[2 * q + 1].y);
}

// Dynamic warp tasks (a.dyn): the first GW tasks go to the warps in order, every later one to the
// warp that claims it from task_ctr[0] (one atomic per task, issued at the start of the previous
// task). Rows are visited longest first, so the claims end the launch with all warps finishing
// together instead of the static round-robin's spread (which accumulates up to one longest task
// per pass over the rows). A task's arithmetic does not depend on which warp runs it, so results
// stay bitwise reproducible. The last CTA to finish zeroes the counters for the next launch.
// a.dyn == 2 (A/B): the first task is claimed too, so a CTA that becomes resident late (its SM
// held by a concurrent kernel) does not start one of the longest tasks late
__device__ __forceinline__ int64_t first_task(const SpmmArgs& a, int64_t gw, int lane) {
  if (a.dyn != 2) return gw;
  int c = 0;
  if (lane == 0) c = atomicAdd(a.task_ctr, 1);
  return __shfl_sync(0xffffffffu, c, 0);
}
__device__ __forceinline__ int64_t next_task(const SpmmArgs& a, int64_t t, int64_t GW, int claim) {
  return a.dyn == 2 ? (int64_t)claim : (a.dyn ? GW + claim : t + GW);
}

__device__ __forceinline__ void task_ctr_release(const SpmmArgs& a) {
  if (!a.dyn) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.task_ctr + 1, 1) == (int)gridDim.x - 1) {
      a.task_ctr[0] = 0;
      a.task_ctr[1] = 0;
      __threadfence();
    }
  }
}

// Full-warp kernel (f > 64): chunk = up to 64 float4 (256 columns), lane owns c4 and c4 + 32.
// MINB resident 8-warp CTAs per SM: 3 (80 registers per thread, a few spill bytes) keeps more
// gathers in flight on large problems (config 5 2.973 -> 2.945 ms, config 3 0.619 -> 0.594 ms);
// 2 (128 registers) wins when a warp gets fewer than ~6 light tasks (config 2 SpMM 35 vs 39 µs,
// config 1). profiles/r01_spmm_occupancy_ab.txt.
template <int MINB, bool W256, int UU = U>
__global__ void __launch_bounds__(kThreads, MINB) k_spmm_wide(SpmmArgs a) {
  __shared__ __align__(16) int2 stage[kWarps][40];
  __shared__ float4 part[kRing][kWarps][32 * V];  // heavy rows: per-warp partial sums, kRing tasks deep
  __shared__ int ring_arrive[kRing];              // warps that have written a slot's partials
  __shared__ int ring_gen[kRing];                 // reductions completed per slot (slot reuse)
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x < kRing) {
    ring_arrive[threadIdx.x] = 0;
    ring_gen[threadIdx.x] = 0;
  }
  __syncthreads();
  // heavy rows for this launch: degree buckets >= heavy_bucket (perm leads with them); the warp
  // segments (htask, built by normalize) cover exactly the rows of deg' >= kHeavyMinDeg
  const bool segs = a.hseg == 1 || (a.hseg == 2 && *a.n_mega_ptr > 0);
  const int hbkt = segs ? 32 - __clz(kHeavyMinDeg) : a.heavy_bucket;
  int n_heavy;
  {
    const int c = lane < kBins && lane >= hbkt ? a.bucket_counts[lane] : 0;
    n_heavy = __reduce_add_sync(0xffffffffu, c);
  }
  const int n_light = a.n - n_heavy;
  int2* st = stage[warp];

  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t GW = (int64_t)gridDim.x * kWarps;
  if (segs) {
    // One warp task per (heavy-row segment | light row, chunk), chunk-major, the segments (each
    // <= kHSeg neighbors, the longest tasks) first, then the light rows by descending degree.
    // A heavy row's segments write their partial sums to the workspace; the row's last segment
    // to arrive (per-(row, chunk) counter) adds the partials in segment order and runs the
    // epilogue -- deterministic, and no CTA barrier anywhere (a CTA-split row of degree 260
    // gathers 14 % (f = 1024) / 25 % (f = 200) slower than a degree-250 row handled by one warp;
    // as two segments it recovers a third to half of that: tools/spmm_degree_bench.py).
    const int hs = *a.n_hseg_ptr;
    const int64_t per = (int64_t)hs + n_light;
    const int64_t L = per * a.nchunks;
    for (int64_t t = first_task(a, gw, lane); t < L;) {
      int claim = 0;  // the next task, claimed now so the atomic's round trip hides behind this one
      if (a.dyn && lane == 0) claim = atomicAdd(a.task_ctr, 1);
      const int64_t t_next = next_task(a, t, GW, __shfl_sync(0xffffffffu, claim, 0));
      const int chunk = (int)(t / per);
      const int r = (int)(t % per);
      const int c0 = chunk * a.cw, lim = min(a.f4, c0 + a.cw);
      int row, b, e, first = -1, cnt = 1;
      if (r < hs) {
        const int4 ht = __ldg(a.htask + r);
        row = ht.x; b = ht.y; e = ht.z; first = ht.w;
        cnt = __ldg(a.hcount + first);
      } else {
        row = a.perm[n_heavy + (r - hs)];
        b = a.rowptr[row];
        e = a.rowptr[row + 1];
      }
      uint32_t mw0 = 0, mw1 = 0;  // gate words, loaded before the gathers
      if (a.mbits) {
        const uint32_t* mr = a.mbits + (int64_t)row * a.ldmb;
        const int g0 = W256 ? c0 + 2 * lane : c0 + lane;
        if (g0 < lim) mw0 = __ldg(mr + (g0 >> 3));
        if (!W256 && g0 + 32 < lim) mw1 = __ldg(mr + ((g0 + 32) >> 3));
      }
      int c4, c4b;
      Acc A;
      if (W256) {
        c4 = c0 + 2 * lane;
        c4b = c4 + 1;
        gather256<UU>(a, st, b, e, chunk, c0, lim, lane, A);
      } else {
        c4 = c0 + lane;
        c4b = c4 + 32;
        if (a.cw == 32 * V && lim == (chunk + 1) * a.cw)
          warp_row_sum<true>(a, st, b, e, 16u * c4, 16u * (c4 + 32), lane, A);
        else
          warp_row_sum<false>(a, st, b, e, 16u * min(c4, lim - 1), 16u * min(c4 + 32, lim - 1), lane, A);
      }
      const bool act0 = c4 < lim, act1 = c4b < lim;
      t = t_next;
      if (cnt == 1) {
        if (act0) store_row(a, row, c4, acc_part(A, 0), &mw0);
        if (act1) store_row(a, row, c4b, acc_part(A, 1), W256 ? &mw0 : &mw1);
        continue;
      }
      float4* ws = a.hseg_ws + (int64_t)r * a.f4;
      if (act0) __stcg(ws + c4, acc_part(A, 0));
      if (act1) __stcg(ws + c4b, acc_part(A, 1));
      __threadfence();
      __syncwarp();
      int prev = 0;
      if (lane == 0) prev = atomicAdd(a.hseg_ctr + (int64_t)first * a.nchunks + chunk, 1);
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if (prev == cnt - 1) {  // the row's last segment: combine in segment order
        __threadfence();
        const float4* w0 = a.hseg_ws + (int64_t)first * a.f4;
        if (act0) {
          float4 tot = __ldcg(w0 + c4);
          for (int g = 1; g < cnt; g++) {
            const float4 p = __ldcg(w0 + (int64_t)g * a.f4 + c4);
            tot.x += p.x; tot.y += p.y; tot.z += p.z; tot.w += p.w;
          }
          store_row(a, row, c4, tot, &mw0);
        }
        if (act1) {
          float4 tot = __ldcg(w0 + c4b);
          for (int g = 1; g < cnt; g++) {
            const float4 p = __ldcg(w0 + (int64_t)g * a.f4 + c4b);
            tot.x += p.x; tot.y += p.y; tot.z += p.z; tot.w += p.w;
          }
          store_row(a, row, c4b, tot, W256 ? &mw0 : &mw1);
        }
        if (lane == 0) a.hseg_ctr[(int64_t)first * a.nchunks + chunk] = 0;  // ready for the next launch
      }
    }
    task_ctr_release(a);
    return;
  }

  // ---- phase 1: heavy rows, one CTA per (row, chunk), neighbors split across 8 warps; the
  // mega rows (deg' >= kMegaMinDeg, the first n_mega of perm) additionally split over kMegaSegs
  // CTAs per chunk: each writes its CTA-reduced partial to the workspace and the last of the
  // row's segments to arrive (per-(row, chunk) counter) sums them in segment order and stores
  // (deterministic) -- a 4.5K-degree row no longer serializes ~560 neighbors per warp.
  // No CTA barrier per task: every warp writes its partial sums into the task's ring slot and the
  // LAST warp to arrive (shared-memory counter) reduces them in warp order -- the same fixed
  // order as a barrier-synchronized reduction -- while the other warps go on to their next task
  // (a slot is reused kRing tasks later, once its reduction has released it).
  const int n_mega = min(min(*a.n_mega_ptr, a.cap_mega), n_heavy);
  const int64_t HM = (int64_t)n_mega * kMegaSegs * a.nchunks;
  const int64_t H = HM + (int64_t)(n_heavy - n_mega) * a.nchunks;
  int task_i = 0;
  for (int64_t t = blockIdx.x; t < H; t += gridDim.x, task_i++) {
    const int slot = task_i % kRing, gen = task_i / kRing;
    int chunk, row, sgi = -1, m = 0;
    if (t < HM) {
      chunk = (int)(t / ((int64_t)n_mega * kMegaSegs));
      const int r = (int)(t % ((int64_t)n_mega * kMegaSegs));
      m = r / kMegaSegs;
      sgi = r % kMegaSegs;
      row = a.perm[m];
    } else {
      const int64_t u = t - HM;
      chunk = (int)(u / (n_heavy - n_mega));
      row = a.perm[n_mega + (int)(u % (n_heavy - n_mega))];
    }
    int b = a.rowptr[row], e = a.rowptr[row + 1];
    if (sgi >= 0) {  // this CTA's segment of the mega row
      const int sl = (e - b + kMegaSegs - 1) / kMegaSegs;
      b = min(e, b + sgi * sl);
      e = min(e, b + sl);
    }
    int seg = (e - b + kWarps - 1) / kWarps;
    seg = (seg + a.seg_align - 1) / a.seg_align * a.seg_align;
    const int w0 = min(e, b + warp * seg), w1 = min(e, w0 + seg);
    const int c0 = chunk * a.cw, lim = min(a.f4, c0 + a.cw);
    int c4, c4b;  // output float4 columns of acc_part(A, 0) and acc_part(A, 1)
    Acc A;
    if (W256) {
      c4 = c0 + 2 * lane;
      c4b = c4 + 1;
      gather256<UU>(a, st, w0, w1, chunk, c0, lim, lane, A);
    } else {
      c4 = c0 + lane;
      c4b = c4 + 32;
      if (a.cw == 32 * V && lim == (chunk + 1) * a.cw)
        warp_row_sum<true>(a, st, w0, w1, 16u * c4, 16u * (c4 + 32), lane, A);
      else
        warp_row_sum<false>(a, st, w0, w1, 16u * min(c4, lim - 1), 16u * min(c4 + 32, lim - 1), lane, A);
    }
    const bool act0 = c4 < lim, act1 = c4b < lim;
    while (*reinterpret_cast<volatile int*>(&ring_gen[slot]) < gen) {
    }  // the slot's previous task has been reduced
    part[slot][warp][lane] = acc_part(A, 0);
    part[slot][warp][lane + 32] = acc_part(A, 1);
    __threadfence_block();
    __syncwarp();
    int arrived = 0;
    if (lane == 0) arrived = atomicAdd(&ring_arrive[slot], 1);
    arrived = __shfl_sync(0xffffffffu, arrived, 0);
    if (arrived == kWarps - 1) {  // the last warp of this task reduces it
      __threadfence_block();
      if (lane == 0) ring_arrive[slot] = 0;
      float4 s[V];
#pragma unroll
      for (int q = 0; q < V; q++) {
        s[q] = part[slot][0][lane + 32 * q];
#pragma unroll
        for (int w = 1; w < kWarps; w++) {
          const float4 p = part[slot][w][lane + 32 * q];
          s[q].x += p.x; s[q].y += p.y; s[q].z += p.z; s[q].w += p.w;
        }
      }
      if (sgi < 0) {
#pragma unroll
        for (int q = 0; q < V; q++)
          if (q == 0 ? act0 : act1) store_row(a, row, q == 0 ? c4 : c4b, s[q]);
      } else {
        float4* ws = a.mega_ws + ((int64_t)m * kMegaSegs + sgi) * a.f4;
#pragma unroll
        for (int q = 0; q < V; q++)
          if (q == 0 ? act0 : act1) __stcg(ws + (q == 0 ? c4 : c4b), s[q]);
        __threadfence();
        __syncwarp();
        int prev = 0;
        if (lane == 0) prev = atomicAdd(a.mega_ctr + (int64_t)m * a.nchunks + chunk, 1);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev == kMegaSegs - 1) {  // last segment of this (row, chunk): combine in order
          __threadfence();
#pragma unroll
          for (int q = 0; q < V; q++) {
            const int cq = q == 0 ? c4 : c4b;
            if (!(q == 0 ? act0 : act1)) continue;
            float4 tot = __ldcg(a.mega_ws + (int64_t)m * kMegaSegs * a.f4 + cq);
            for (int g = 1; g < kMegaSegs; g++) {
              const float4 p = __ldcg(a.mega_ws + ((int64_t)m * kMegaSegs + g) * a.f4 + cq);
              tot.x += p.x; tot.y += p.y; tot.z += p.z; tot.w += p.w;
            }
            store_row(a, row, cq, tot);
          }
          if (lane == 0) a.mega_ctr[(int64_t)m * a.nchunks + chunk] = 0;  // ready for the next launch
        }
      }
      __threadfence_block();
      __syncwarp();
      if (lane == 0) *reinterpret_cast<volatile int*>(&ring_gen[slot]) = gen + 1;  // release the slot
    }
  }

  // ---- phase 2: light rows, one warp per (row, chunk) ----
  const int64_t L = (int64_t)n_light * a.nchunks;
  for (int64_t t = first_task(a, gw, lane); t < L;) {
    int claim = 0;
    if (a.dyn && lane == 0) claim = atomicAdd(a.task_ctr, 1);
    const int64_t t_next = next_task(a, t, GW, __shfl_sync(0xffffffffu, claim, 0));
    const int chunk = (int)(t / n_light);
    const int row = a.perm[n_heavy + (int)(t % n_light)];
    const int c0 = chunk * a.cw, lim = min(a.f4, c0 + a.cw);
    const int b = a.rowptr[row], e = a.rowptr[row + 1];
    int c4, c4b;
    // the gate word is loaded before the gathers (its latency hides behind them) instead of
    // after them, where it would add a dependent round trip to every task
    uint32_t mw0 = 0, mw1 = 0;
    if (a.mbits) {
      const uint32_t* mr = a.mbits + (int64_t)row * a.ldmb;
      const int g0 = W256 ? c0 + 2 * lane : c0 + lane;
      if (g0 < lim) mw0 = __ldg(mr + (g0 >> 3));
      if (!W256 && g0 + 32 < lim) mw1 = __ldg(mr + ((g0 + 32) >> 3));
    }
    Acc A;
    if (W256) {
      c4 = c0 + 2 * lane;
      c4b = c4 + 1;
      gather256<UU>(a, st, b, e, chunk, c0, lim, lane, A);
    } else {
      c4 = c0 + lane;
      c4b = c4 + 32;
      if (a.cw == 32 * V && lim == (chunk + 1) * a.cw)
        warp_row_sum<true>(a, st, b, e, 16u * c4, 16u * (c4 + 32), lane, A);
      else
        warp_row_sum<false>(a, st, b, e, 16u * min(c4, lim - 1), 16u * min(c4 + 32, lim - 1), lane, A);
    }
    if (c4 < lim) store_row(a, row, c4, acc_part(A, 0), &mw0);
    if (c4b < lim) store_row(a, row, c4b, acc_part(A, 1), W256 ? &mw0 : &mw1);
    t = t_next;
  }
  task_ctr_release(a);
}

// Sub-warp kernel (f <= 64): groups of G lanes, one row per group; heavy rows CTA-split.
// Rows with deg' >= kNarrowSplitDeg (the first rows of the degree-sorted order, whole degree
// buckets, at most two per CTA) are split over all NG = 8 * 32/G lane groups of a CTA and reduced through shared memory
// in group order; every other row is one group's. (At f <= 64 a row costs one dependent round
// trip per 8 neighbors, so a 170-degree row alone would otherwise set the kernel's length.)
constexpr int kNarrowSplitDeg = 64;
template <int G>
__global__ void __launch_bounds__(kThreads) k_spmm_narrow(SpmmArgs a) {
  constexpr int PER = 32 / G;
  constexpr int NG = kWarps * PER;
  __shared__ float4 part[NG][G];
  __shared__ int s_nh;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int g = lane / G, gl = lane % G;
  const int gi = warp * PER + g;
  if (threadIdx.x == 0) {
    // at most two split rows per CTA: enough to cut the critical path of a few outlier rows
    // without serializing a batch's many medium rows. The split set is whole degree buckets,
    // highest first (perm leads with them), so it depends only on the degree histogram and
    // not on the (atomic) order of rows inside a bucket: every row's summation order is fixed
    // and the result is bitwise reproducible (R14).
    const int cap = 2 * (int)gridDim.x;
    int h = 0;
    for (int bkt = kBins - 1; bkt >= 32 - __clz(kNarrowSplitDeg); bkt--) {
      const int c = a.bucket_counts[bkt];
      if (h + c > cap) break;
      h += c;
    }
    s_nh = h;
  }
  __syncthreads();
  const int n_split = s_nh;
  const int n_rest = a.n - n_split;
  const bool act = gl < a.f4;
  for (int64_t t = blockIdx.x; t < n_split; t += gridDim.x) {
    const int row = a.perm[t];
    const int b = a.rowptr[row], e = a.rowptr[row + 1];
    const int seg = (e - b + NG - 1) / NG;
    const int w0 = min(e, b + gi * seg), w1 = min(e, w0 + seg);
    part[gi][gl] = group_row_sum(a, w0, w1, gl, act);
    __syncthreads();
    if (threadIdx.x < G) {
      float4 s4 = part[0][threadIdx.x];
#pragma unroll 4
      for (int q = 1; q < NG; q++) {
        const float4 p = part[q][threadIdx.x];
        s4.x += p.x; s4.y += p.y; s4.z += p.z; s4.w += p.w;
      }
      if ((int)threadIdx.x < a.f4) store_row(a, row, threadIdx.x, s4);
    }
    __syncthreads();
  }
  const int64_t gid = ((int64_t)blockIdx.x * kWarps + warp) * PER + g;
  const int64_t GN = (int64_t)gridDim.x * kWarps * PER;
  for (int64_t t = gid; t < n_rest; t += GN) {
    const int row = a.perm[n_split + (int)t];
    const float4 acc = group_row_sum(a, a.rowptr[row], a.rowptr[row + 1], gl, act);
    if (act) store_row(a, row, gl, acc);
  }
}

template <typename K>
int launch_k(gsg_ctx* ctx, K kern, std::atomic<int>* occ_cache, const SpmmArgs& a, int64_t warp_tasks) {
  int occ = occ_cache->load(std::memory_order_relaxed);
  if (occ < 1) {  // resident CTAs per SM (the same on every sm_100a device this library accepts)
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, 0) != cudaSuccess || occ < 1) occ = 1;
    occ_cache->store(occ, std::memory_order_relaxed);
  }
  int64_t want = (warp_tasks + kWarps - 1) / kWarps;
  int64_t grid = (int64_t)ctx->num_sms * occ;
  if (want < grid) grid = want;
  if (grid < 1) grid = 1;
  kern<<<(int)grid, kThreads, 0, ctx->stream>>>(a);
  count_launch(ctx);
  GSG_CUDA(cudaGetLastError());
  return GSG_OK;
}

}  // namespace

int spmm_launch(gsg_ctx* ctx, const gsg_subgraph* sg, int transpose, int f, const float* X, int64_t ldx,
                float* Y, int64_t ldy, void* Ylp, int64_t ldylp, const float* mask, int64_t ldm, int relu,
                int accum, const BitsIO& bits) {
  GSG_CHECK(sg->norm_mode >= 0, GSG_EINVAL, "subgraph not normalized (call gsg_subgraph_normalize)");
  GSG_CHECK(f >= 1, GSG_EINVAL, "f must be >= 1 (got %d)", f);
  if (sg->n == 0) return GSG_OK;
  GSG_CHECK(X && Y, GSG_EINVAL, "X and Y must be non-NULL");
  GSG_CHECK(ldx >= f && ldx % 4 == 0, GSG_EINVAL, "ldx=%lld must be >= f=%d and a multiple of 4", (long long)ldx, f);
  GSG_CHECK(ldy >= f && ldy % 4 == 0, GSG_EINVAL, "ldy=%lld must be >= f=%d and a multiple of 4", (long long)ldy, f);
  GSG_CHECK(((uintptr_t)X | (uintptr_t)Y) % 16 == 0, GSG_EINVAL, "X/Y must be 16-byte aligned");
  GSG_CHECK(!Ylp || (ldylp >= f && ldylp % 8 == 0 && (uintptr_t)Ylp % 16 == 0), GSG_EINVAL,
            "bf16 output needs ldylp >= f, ldylp %% 8 == 0 and 16-byte alignment");
  GSG_CHECK(!mask || (ldm >= f && ldm % 4 == 0 && (uintptr_t)mask % 16 == 0), GSG_EINVAL,
            "mask needs ldm >= f, ldm %% 4 == 0 and 16-byte alignment");
  GSG_CHECK(X != Y, GSG_EINVAL, "Y must not alias X");
  const int64_t nwords = (f + 31) / 32;
  GSG_CHECK(!bits.in || (bits.ldi >= nwords && (uintptr_t)bits.in % 4 == 0), GSG_EINVAL,
            "bitmask gate needs ldmb >= ceil(f/32) (ldmb=%lld)", (long long)bits.ldi);
  GSG_CHECK(!bits.out || (relu && bits.ldo >= nwords && (uintptr_t)bits.out % 4 == 0), GSG_EINVAL,
            "bitmask output needs the ReLU epilogue and ldob >= ceil(f/32)");
  GSG_CHECK((int64_t)sg->n * ldx * 4 < ((int64_t)1 << 32), GSG_EUNSUPPORTED,
            "X too large for 32-bit byte offsets (n * ldx * 4 >= 4 GiB)");
  // algorithmic (effective gather) bytes, SURVEY §8(d)
  const double nh = (double)sg->nnz_hat, nn = (double)sg->n;
  ProfScope ps(ctx, GSG_K_SPMM, 4.0 * nh * f + 8.0 * nh + 4.0 * (nn + 1) + 4.0 * nn * f, 2.0 * nh * f);
  SpmmArgs a{};
  a.n = sg->n;
  a.f4 = (f + 3) / 4;
  a.rowptr = sg->rowptr;
  a.col = sg->col;
  a.val = transpose ? sg->valT : sg->val;
  a.X = reinterpret_cast<const float4*>(X);
  a.ldx4 = (uint32_t)(ldx / 4);
  a.ldx16 = (uint32_t)(ldx * 4);
  a.Y = reinterpret_cast<float4*>(Y);
  a.ldy4 = ldy / 4;
  a.Ylp = reinterpret_cast<uint2*>(Ylp);
  a.ldylp4 = ldylp / 4;
  a.mask = bits.in ? nullptr : reinterpret_cast<const float4*>(mask);
  a.mbits = bits.in;
  a.ldmb = bits.ldi;
  a.obits = bits.out;
  a.ldob = bits.ldo;
  a.f = f;
  if (bits.out) GSG_CUDA(cudaMemset2DAsync(bits.out, bits.ldo * 4, 0, nwords * 4, sg->n, ctx->stream));
  a.relu = relu;
  a.accum = accum;
  a.ldm4 = ldm / 4;
  a.perm = sg->perm;
  a.n_heavy_ptr = sg->counters + kBins;
  a.bucket_counts = sg->counters;
  a.n_mega_ptr = sg->counters + kNMega;
  static std::atomic<int> occ_wide{0}, occ_wide3{0}, occ_widen{0}, occ_wide3n{0}, occ16{0}, occ8{0}, occ4{0};
  if (a.f4 > 16) {
    a.nchunks = (a.f4 + 32 * V - 1) / (32 * V);
    {  // mega-row workspace: at most nnz' / kMegaMinDeg rows can have deg' >= kMegaMinDeg
      const int cap = (int)std::min<int64_t>(sg->n, sg->nnz_hat / kMegaMinDeg);
      a.cap_mega = cap;
      if (cap > 0) {
        const int nch = a.nchunks;
        if (int rc = ctx->ws_mega.reserve(sizeof(float4) * (size_t)cap * kMegaSegs * a.f4)) return rc;
        // a grown buffer is zeroed whole (cudaMalloc may hand back the old address, so growth,
        // not a pointer change, is the test); afterwards every launch leaves the counters at zero
        const size_t had = ctx->ws_megactr.bytes;
        if (int rc = ctx->ws_megactr.reserve(sizeof(int) * (size_t)cap * std::max(nch, 16))) return rc;
        if (ctx->ws_megactr.bytes != had) GSG_CUDA(cudaMemsetAsync(ctx->ws_megactr.ptr, 0, ctx->ws_megactr.bytes, ctx->stream));
        a.mega_ws = static_cast<float4*>(ctx->ws_mega.ptr);
        a.mega_ctr = static_cast<int*>(ctx->ws_megactr.ptr);
      }
    }
    // heavy rows as warp segments (GSG_SPMM_HSEG=0: the CTA-split heavy phase, A/B)
    static const int hseg_env = getenv("GSG_SPMM_HSEG") ? atoi(getenv("GSG_SPMM_HSEG")) : 1;
    // Warp segments beat CTA-split heavy rows for narrow launches (f <= 512: config 3-5 f = 200
    // 36.2 -> 33.0 / 50.8 -> 48.2 / 120.6 -> 116.8 us) and where mega rows exist (config 4
    // f = 1024 180 -> 166 us), but not for the f = 1024 launches of graphs without them (config 5
    // 522 -> 529, config 3 107 -> 109 us): hseg = 2 lets the kernel decide from the device-side
    // mega-row count. profiles/r02_spmm_hseg_ab.txt
    static const int hb_env = getenv("GSG_SPMM_HEAVY_BUCKET") ? atoi(getenv("GSG_SPMM_HEAVY_BUCKET")) : 0;  // A/B
    a.heavy_bucket = hb_env > 0 ? hb_env : 32 - __builtin_clz((unsigned)kHeavyMinDeg);
    // a CTA-split row's per-warp shares in multiples of 8 neighbors (one batch): no partial batch
    // inside a row; the last warps take the remainder, and with no barrier per task an idle warp
    // moves on (config 5 f = 1024 515.7 -> 510.4 us; 32 slower; profiles/r02_spmm_heavy_ring_ab.txt)
    static const int align_env = getenv("GSG_SPMM_SEG_ALIGN") ? atoi(getenv("GSG_SPMM_SEG_ALIGN")) : 8;
    a.seg_align = std::max(1, align_env);
    // GSG_SPMM_HSEG (A/B): 0 never, 2 always, 3 only where mega rows exist (at every width)
    a.hseg = (hseg_env && sg->htask) ? (hseg_env == 2 || (hseg_env == 1 && a.nchunks < 4) ? 1 : 2) : 0;
    if (a.hseg) {
      const size_t cap = sg->cap_hseg;
      if (int rc = ctx->ws_hseg.reserve(sizeof(float4) * cap * a.f4)) return rc;
      const size_t had = ctx->ws_hsegctr.bytes;
      if (int rc = ctx->ws_hsegctr.reserve(sizeof(int) * cap * a.nchunks)) return rc;
      if (ctx->ws_hsegctr.bytes != had)
        GSG_CUDA(cudaMemsetAsync(ctx->ws_hsegctr.ptr, 0, ctx->ws_hsegctr.bytes, ctx->stream));
      a.htask = sg->htask;
      a.hcount = sg->hcount;
      a.n_hseg_ptr = sg->counters + kNHSeg;
      a.hseg_ws = static_cast<float4*>(ctx->ws_hseg.ptr);
      a.hseg_ctr = static_cast<int*>(ctx->ws_hsegctr.ptr);
    }
    static const int dyn_env = getenv("GSG_SPMM_DYN") ? atoi(getenv("GSG_SPMM_DYN")) : 1;  // A/B: 0 static
    a.dyn = dyn_env == 2 ? 2 : (dyn_env ? 1 : 0);
    if (a.dyn) {
      const size_t had = ctx->ws_taskctr.bytes;
      if (int rc = ctx->ws_taskctr.reserve(2 * sizeof(int))) return rc;
      if (ctx->ws_taskctr.bytes != had) GSG_CUDA(cudaMemsetAsync(ctx->ws_taskctr.ptr, 0, ctx->ws_taskctr.bytes, ctx->stream));
      a.task_ctr = static_cast<int*>(ctx->ws_taskctr.ptr);
    }
    a.cw = (a.f4 + a.nchunks - 1) / a.nchunks;
    static const int w256_env = getenv("GSG_SPMM_W256") ? atoi(getenv("GSG_SPMM_W256")) : 1;
    a.w256 = w256_env && (uintptr_t)X % 32 == 0 && ldx % 8 == 0;  // GSG_SPMM_W256=0: 128-bit path (A/B)
    if (a.w256) a.cw = (a.cw + 1) & ~1;  // chunks start on 32-byte column pairs
    // a narrow remainder (r = f4 mod 64 <= 32 float4 past whole 64-float4 chunks) as its own chunk
    // gathered by lane groups (warp_row_sum256_grp) instead of equal chunks with idle lanes:
    // f = 300 -> 64 + 11 float4 (1.25 load instructions per neighbor instead of 2), f = 602 ->
    // 64 + 64 + 23 (2.5 instead of 3). GSG_SPMM_TAIL=0 keeps equal chunks (A/B).
    static const int tail_env = getenv("GSG_SPMM_TAIL") ? atoi(getenv("GSG_SPMM_TAIL")) : 1;
    a.tailg = 0;
    {
      const int r = a.f4 % (32 * V);
      if (tail_env && a.w256 && a.f4 > 32 * V && r > 0 && r <= 32) {
        a.cw = 32 * V;
        a.tailg = r <= 16 ? 8 : 16;
      }
    }
    const int64_t tasks = (int64_t)sg->n * a.nchunks;
    static const int minb_env = getenv("GSG_SPMM_MINB") ? atoi(getenv("GSG_SPMM_MINB")) : 0;  // A/B: force 2 or 3
    // (static schedule: three CTAs per SM from ~4 (row, chunk) tasks per warp on -- config 5 / 4
    // f = 200 125.5 -> 119.9 / 52.6 -> 50.8 us; profiles/r02_spmm_variants_ab.txt)
    // With dynamically claimed tasks (a.dyn) two CTAs/SM (128 registers) gather as fast or faster
    // on launches of one or two column chunks (f <= 512: config 5 f = 200 111.0 -> 109.5 us alone,
    // config 3 f = 512 56.8 -> 53.0; steps: config 2 0.480 -> 0.463 ms, config 3 0.552 -> 0.531,
    // config 5 2.787 -> 2.785), except for the lane-group remainder launches (f = 300 168.8 ->
    // 176.0 at two); the 4-chunk f = 1024 launches keep three (in-step neutral to slightly worse
    // at two). profiles/r02_spmm_occupancy_dyn_ab.txt. GSG_SPMM_OCC_RULE (A/B): 0 the
    // static-schedule rule (three from ~4 tasks per warp on), 1 two for every non-remainder launch.
    static const int occ_rule = getenv("GSG_SPMM_OCC_RULE") ? atoi(getenv("GSG_SPMM_OCC_RULE")) : 2;
    const bool many = tasks >= 4LL * ctx->num_sms * 3 * kWarps;
    const bool two_ok = a.dyn && !a.tailg && (occ_rule == 1 || (occ_rule == 2 && a.nchunks <= 2));
    const bool three = minb_env == 3 || (minb_env != 2 && many && !two_ok);
    static const int u_env = getenv("GSG_SPMM_U") ? atoi(getenv("GSG_SPMM_U")) : 8;  // A/B: gathers in flight
    static std::atomic<int> occ36{0}, occ44{0};
    if (a.w256 && minb_env == 4) return launch_k(ctx, k_spmm_wide<4, true, 4>, &occ44, a, tasks);
    if (a.w256 && three && u_env == 6) return launch_k(ctx, k_spmm_wide<3, true, 6>, &occ36, a, tasks);
    if (a.w256)
      return three ? launch_k(ctx, k_spmm_wide<3, true>, &occ_wide3, a, tasks)
                   : launch_k(ctx, k_spmm_wide<2, true>, &occ_wide, a, tasks);
    return three ? launch_k(ctx, k_spmm_wide<3, false>, &occ_wide3n, a, tasks)
                 : launch_k(ctx, k_spmm_wide<2, false>, &occ_widen, a, tasks);
  }
  a.nchunks = 1;
  a.cw = a.f4;
  if (a.f4 > 8) return launch_k(ctx, k_spmm_narrow<16>, &occ16, a, (int64_t)sg->n / 2 + 1);
  if (a.f4 > 4) return launch_k(ctx, k_spmm_narrow<8>, &occ8, a, (int64_t)sg->n / 4 + 1);
  return launch_k(ctx, k_spmm_narrow<4>, &occ4, a, (int64_t)sg->n / 8 + 1);
}

}  // namespace gsg
