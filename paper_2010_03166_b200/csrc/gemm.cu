// gemm.cu -- SURVEY §8(a) rows a3 (H = ReLU(P W)), a5 (dW = Pᵀ dZ), a6 (T = dZ Wᵀ) and the
// head GEMMs: the paper's "weight transformation" (MKL cblas_dgemm at P:1204),
// re-designed as a warp-specialized tcgen05 kernel for sm_100a:
//   warp 0        TMA producer  (cp.async.bulk.tensor, 128B swizzle, S-stage smem ring)
//   warp 1        MMA issuer    (one thread issues tcgen05.mma kind::tf32 / kind::f16,
//                                M=128, N=BN, accumulators in TMEM)
//   warp 2        TMEM allocator (2 x BN fp32 accumulator columns: double-buffered tiles)
//   warps 4..7    epilogue      (tcgen05.ld 32x32b -> ReLU / ReLU'-mask / split-K partial ->
//                                global stores, optional bf16 copy)
// Persistent grid over (m-block, n-block, k-split) tiles. Operands are read straight from the
// row-major activations: K-major (A = P or dZ; B = Wᵀ) or MN-major (A = Pᵀ, B = W or dZ)
// shared-memory descriptors, so no transposed copies are ever materialized.
// Split-K partials are reduced in a fixed split order (bitwise reproducible).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include <atomic>

#include "common.cuh"

namespace gsg {
namespace {

constexpr int BM = 128;
// warps 0-3: TMA producer, MMA issuer, TMEM allocator, idle; warps 4-11: epilogue. Two epilogue
// warps per TMEM lane quarter, each taking half of the tile's columns: the epilogue is bound by
// its per-warp instruction latency (measured: a K = 64 GEMM spends 2/3 of its time there).
constexpr int kEpiWarps = 8;
constexpr int kGemmThreads = 128 + 32 * kEpiWarps;

// ------------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
template <bool BF16>
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  if constexpr (BF16) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
  }
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor (sm_100 version bits). layout: 2 = SWIZZLE_128B (16-byte
// granules, 8-row atoms), 1 = SWIZZLE_128B_BASE32B (32-byte granules, 4-row atoms) -- the only
// layout tcgen05 accepts for MN-major 32-bit (tf32) operands.
template <int LAYOUT = 2>
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)LAYOUT << 61);
}

// MN-major operand descriptor for k-step kk: MN blocks of 128 B at stride BK*128 (LBO);
// bf16: 8-row SW128 atoms (SBO 1024), tf32: 4-row SW128_BASE32B atoms (SBO 512). One k-step
// covers UMMA_K rows of 128 B = 1024 B (tf32, 8 rows) or 2048 B (bf16, 16 rows).
template <bool BF16, int BK>
__device__ __forceinline__ uint64_t mn_desc(uint32_t base, int kk) {
  if constexpr (BF16) return smem_desc<2>(base + kk * 2048, BK * 128, 1024);
  else return smem_desc<1>(base + kk * 1024, BK * 128, 512);
}

struct GemmArgs {
  int M, N, K;
  int num_m, num_n, splits, kb_per_split, num_kb;
  float* C;
  int64_t ldc;
  __nv_bfloat16* Clp;
  int64_t ldclp;
  const float* aux;
  int64_t ldaux;
  int epi;          // GSG_EPI_*
  int accumulate;
  float* ws;        // split-K partials [splits][M][ldws]
  int64_t ldws;
  int mpad;         // rows per split in ws (num_m * tile rows): TMA-stored partial tiles never straddle splits
  int tma_store;    // 1: C / ws written by TMA bulk-tensor stores from swizzled smem staging
  int aux_tma;      // 1: the GSG_EPI_MASK operand is fetched by TMA (tmX) into the staging buffer
  const uint32_t* abits;  // GSG_EPI_MASK gate as a ReLU bitmask (gsg.h "ReLU bitmask") instead of aux
  int64_t ldab;
  uint32_t* cbits;        // GSG_EPI_RELU: also write the bitmask 1[C > 0] (splits == 1 only)
  int64_t ldcb;
  uint32_t idesc;
  int x3nkb;        // FP32X3 with implicit hi: k-blocks per segment of K' = [A | A | A_lo] x [B ; B_lo ; B] (0: off)
  int x3dual;       // k_gemm_x3: each tile's K piece split over both TMEM accumulators (pieces > 32 k-blocks)
};

// 1[x_i > 0] of one 32-column epilogue chunk (col0 % 32 == 0) as a bitmask word; columns past
// N (valid < 32) are cleared.
// Two instructions per element: the sign bit of 0 - x (round-to-nearest: +0 for x = +-0, negative
// iff x > 0) is funnel-shifted into the word, column 31 first.
__device__ __forceinline__ uint32_t relu_bits(const float (&x)[32], int valid) {
  uint32_t b = 0;
#pragma unroll
  for (int i = 31; i >= 0; i--) b = __funnelshift_l(__float_as_uint(__fsub_rn(0.f, x[i])), b, 1);
  return valid >= 32 ? b : b & ((1u << valid) - 1u);
}

// wb[i] = w without dynamic register-array indexing (i < 4)
__device__ __forceinline__ void set_word(uint32_t (&wb)[4], int i, uint32_t w) {
  wb[0] = i == 0 ? w : wb[0];
  wb[1] = i == 1 ? w : wb[1];
  wb[2] = i == 2 ? w : wb[2];
  wb[3] = i == 3 ? w : wb[3];
}

// The CPW bitmask words of one row that one epilogue warp produced for a tile (word w0 = first
// chunk's column / 32): one 16- (8-) byte store per lane when they are all inside the row's
// ceil(N/32) words and aligned, else one store per valid word.
template <int CPW>
__device__ __forceinline__ void store_words(const GemmArgs& g, int row, int w0, const uint32_t (&wb)[4]) {
  uint32_t* p = g.cbits + (int64_t)row * g.ldcb + w0;
  const int nw = (g.N + 31) >> 5;
  if (w0 + CPW <= nw && ((uintptr_t)p % (4 * CPW)) == 0) {
    if constexpr (CPW == 4) *reinterpret_cast<uint4*>(p) = make_uint4(wb[0], wb[1], wb[2], wb[3]);
    else if constexpr (CPW == 2) *reinterpret_cast<uint2*>(p) = make_uint2(wb[0], wb[1]);
    else {
#pragma unroll
      for (int i = 0; i < CPW; i++) p[i] = wb[i];
    }
  } else {
#pragma unroll
    for (int i = 0; i < CPW; i++) if (w0 + i < nw) p[i] = wb[i];
  }
}

// x_i = x_i * bit i of the gate word (ReLU' from a bitmask)
__device__ __forceinline__ void gate_bits(float (&x)[32], uint32_t m) {
#pragma unroll
  for (int i = 0; i < 32; i++) x[i] = (m >> i) & 1u ? x[i] : 0.f;
}

// Per-CTA configuration. CTA2 = cta_group::2: a CTA pair computes a 256 x BN tile with one
// tcgen05.mma (M = 256); each CTA stages its 128 rows of A and half (BN/2) of B, so per-SM
// operand traffic per FLOP drops by a third vs. the 128 x BN single-CTA tile.
template <int BN, bool BF16, bool CTA2>
struct Cfg {
  static constexpr int ELEM = BF16 ? 2 : 4;
  static constexpr int BK = 128 / ELEM;             // one 128-byte swizzle row of K
  static constexpr int UMMA_K = 32 / ELEM;          // 8 (tf32) / 16 (bf16)
  static constexpr int MN_PER_ROW = 128 / ELEM;     // MN elements per 128B row (MN-major)
  static constexpr int BMT = CTA2 ? 2 * BM : BM;    // tile rows (M) per CTA group
  static constexpr int BNC = CTA2 ? BN / 2 : BN;    // B rows (N) staged per CTA
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = BNC * 128;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STG = 1;                     // staging buffers per epilogue warp
  // as many operand stages as fit next to the staging buffers (cap 8)
  static constexpr int STAGES_FIT = (232448 - 1280 - kEpiWarps * STG * 4096) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int TMEM_COLS = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  static constexpr int STG_BYTES = kEpiWarps * STG * 4096;  // per epilogue warp: STG x (32 x 32 fp32)
  static constexpr int SMEM = 1024 /*align slack*/ + STAGES * STAGE_BYTES + STG_BYTES + 256 /*barriers*/;
  static_assert(SMEM <= 232448, "GEMM smem over the 227 KB per-CTA limit");
  static_assert(STAGES * 16 + 4 * 8 + kEpiWarps * 8 + 4 <= 256, "GEMM barriers overflow their 256 B");
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Arrive on the pair leader's barrier. Default (.release.cta) semantics: only the TMEM reads must
// be ordered before it, and tcgen05.fence::before_thread_sync does that. An explicit .release.cluster
// compiles to MEMBAR.ALL.GPU + ERRBAR, which drains this thread's outstanding TMA stores every tile.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA load whose completion is counted on the pair leader's mbarrier (cta_group::2)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
template <bool BF16>
__device__ __forceinline__ void tc_mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  if constexpr (BF16) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
  }
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

// The kernel body; the tensor maps are references to the launching kernel's __grid_constant__
// parameters (k_gemm: four maps; k_gemm_x3 adds the two lo operands of an implicit-hi FP32X3
// GEMM, so that plain launches keep their parameter block as it was).
template <int BN, bool BF16, bool A_MN, bool B_MN, bool CTA2, bool X3>
__device__ __forceinline__ void gemm_body(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                                          const CUtensorMap& tmX, const CUtensorMap& tmA2, const CUtensorMap& tmB2,
                                          const GemmArgs& g) {
  using C = Cfg<BN, BF16, CTA2>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = smem + C::STAGES * C::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + C::STG_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* auxbar = tempty + 2;  // [kEpiWarps] one per epilogue warp: TMA loads of the gate operand
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(auxbar + kEpiWarps);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tiles = g.num_m * g.num_n * g.splits;
  const uint32_t rank = CTA2 ? cluster_rank() : 0u;
  const bool leader = rank == 0;
  const int group = CTA2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int ngroups = CTA2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    if constexpr (X3) {
      prefetch_tmap(&tmA2);
      prefetch_tmap(&tmB2);
    }
    if (g.tma_store) prefetch_tmap(&tmC);
    for (int s = 0; s < C::STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; a++) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], CTA2 ? 2 * kEpiWarps : kEpiWarps); }
    for (int w = 0; w < kEpiWarps; w++) mbar_init(&auxbar[w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if constexpr (CTA2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if constexpr (CTA2) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer (both CTAs of a pair) =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = group; t < tiles; t += ngroups) {
        const int per_split = g.num_m * g.num_n;
        const int s = t / per_split, r = t % per_split;
        const int mb = r / g.num_n, nb = r % g.num_n;
        const int m0 = mb * C::BMT + (int)rank * BM;
        const int n0 = nb * BN + (int)rank * C::BNC;
        const int kb0 = s * g.kb_per_split, kb1 = min(g.num_kb, kb0 + g.kb_per_split);
        for (int kb = kb0; kb < kb1; kb++) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          // FP32X3 (implicit hi): k-block kb of segment seg reads A (seg 0, 1) or A_lo (seg 2) and
          // B (seg 0, 2) or B_lo (seg 1) at the segment's own k; each segment's last box is
          // zero-filled by TMA past K
          const CUtensorMap* pA = &tmA;
          const CUtensorMap* pB = &tmB;
          int kk = kb;
          if constexpr (X3) {
            const int seg = kb / g.x3nkb;
            kk = kb - seg * g.x3nkb;
            if (seg == 2) pA = &tmA2;
            if (seg == 1) pB = &tmB2;
          }
          const int k0 = kk * C::BK;
          if constexpr (CTA2) {
            const uint32_t lb = map_to_rank(smem_u32(&full[stage]), 0);
            if (leader) mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            if constexpr (A_MN) {
#pragma unroll
              for (int j = 0; j < BM / C::MN_PER_ROW; j++)
                tma_load_2d_pair(sa + j * (C::BK * 128), pA, lb, m0 + j * C::MN_PER_ROW, k0);
            } else {
              tma_load_2d_pair(sa, pA, lb, k0, m0);
            }
            if constexpr (B_MN) {
#pragma unroll
              for (int j = 0; j < C::BNC / C::MN_PER_ROW; j++)
                tma_load_2d_pair(sb + j * (C::BK * 128), pB, lb, n0 + j * C::MN_PER_ROW, k0);
            } else {
              tma_load_2d_pair(sb, pB, lb, k0, n0);
            }
          } else {
            mbar_expect_tx(&full[stage], C::STAGE_BYTES);
            if constexpr (A_MN) {
#pragma unroll
              for (int j = 0; j < BM / C::MN_PER_ROW; j++)
                tma_load_2d(sa + j * (C::BK * 128), pA, &full[stage], m0 + j * C::MN_PER_ROW, k0);
            } else {
              tma_load_2d(sa, pA, &full[stage], k0, m0);
            }
            if constexpr (B_MN) {
#pragma unroll
              for (int j = 0; j < C::BNC / C::MN_PER_ROW; j++)
                tma_load_2d(sb + j * (C::BK * 128), pB, &full[stage], n0 + j * C::MN_PER_ROW, k0);
            } else {
              tma_load_2d(sb, pB, &full[stage], k0, n0);
            }
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (pair leader only) =====================
    if (lane == 0 && leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = group; t < tiles; t += ngroups) {
        const int per_split = g.num_m * g.num_n;
        const int s = t / per_split;
        const int kb0 = s * g.kb_per_split, kb1 = min(g.num_kb, kb0 + g.kb_per_split);
        // X3 (FP32X3): each tile's K piece in two halves, one per TMEM accumulator (each half
        // <= 32 k-blocks: the accumulator drift bound), added by the epilogue in order -- two
        // pieces per tile without a split-K reduction; both accumulators belong to every tile
        const bool dual = X3 && g.x3dual;
        const int half = dual ? (kb1 - kb0 + 1) / 2 : kb1 - kb0;
        if (dual) {
          mbar_wait(&tempty[0], acc_phase ^ 1);
          mbar_wait(&tempty[1], acc_phase ^ 1);
        } else {
          mbar_wait(&tempty[acc], acc_phase ^ 1);
        }
        tc_fence_after();
        for (int kb = kb0; kb < kb1; kb++) {
          const int ai = dual ? (kb - kb0 >= half ? 1 : 0) : acc;
          const int kstart = dual && ai ? kb0 + half : kb0;
          const uint32_t tmem_d = tmem_base + ai * BN;
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t b_addr = a_addr + C::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < C::BK / C::UMMA_K; kk++) {
            uint64_t ad, bd;
            if constexpr (A_MN) ad = mn_desc<BF16, C::BK>(a_addr, kk);
            else ad = smem_desc<2>(a_addr + kk * 32, 16, 1024);
            if constexpr (B_MN) bd = mn_desc<BF16, C::BK>(b_addr, kk);
            else bd = smem_desc<2>(b_addr + kk * 32, 16, 1024);
            const uint32_t en = (kb > kstart || kk > 0) ? 1u : 0u;
            if constexpr (CTA2) tc_mma_pair<BF16>(tmem_d, ad, bd, g.idesc, en);
            else tc_mma<BF16>(tmem_d, ad, bd, g.idesc, en);
          }
          if constexpr (CTA2) tc_commit_pair(&empty[stage]);
          else tc_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if constexpr (CTA2) tc_commit_pair(&tfull[dual ? 0 : acc]);
        else tc_commit(&tfull[dual ? 0 : acc]);
        if (dual) acc_phase ^= 1;
        else if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue (own 128 rows of the tile) =====================
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    const int e = warp - 4;           // epilogue warp index: staging buffers, aux barrier
    constexpr int CPW = BN / 32 / (kEpiWarps / 4);  // 32-column chunks per warp
    static_assert(CPW >= 1 && CPW <= 4, "bitmask words per warp are kept in uint32_t[4]");
    const int c_begin = (e >> 2) * CPW;
    const uint32_t tempty_leader = CTA2 ? map_to_rank(smem_u32(&tempty[0]), 0) : 0u;
    int sbuf = 0;
    uint32_t aux_phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = group; t < tiles; t += ngroups) {
      const int per_split = g.num_m * g.num_n;
      const int s = t / per_split, r = t % per_split;
      const int mb = r / g.num_n, nb = r % g.num_n;
      const bool dual = X3 && g.x3dual;
      mbar_wait(&tfull[dual ? 0 : acc], acc_phase);
      tc_fence_after();
      bool second = false;  // dual: the tile's second K half sits in accumulator 1
      if (dual) {
        const int kb0 = s * g.kb_per_split, kb1 = min(g.num_kb, kb0 + g.kb_per_split);
        second = kb1 - kb0 > (kb1 - kb0 + 1) / 2;
      }
      const int row_base = mb * C::BMT + (int)rank * BM + q * 32;
      const int row = row_base + lane;
      const bool row_ok = row < g.M;
      uint32_t wb[4] = {0u, 0u, 0u, 0u};  // ReLU bitmask words of this lane's row, one per chunk (cbits)
      for (int c = c_begin; c < c_begin + CPW; c++) {
        uint32_t v[32];
        __syncwarp();
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (dual ? 0 : acc) * BN + c * 32, v);
        if (second) {
          uint32_t v2[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + BN + c * 32, v2);
#pragma unroll
          for (int i = 0; i < 32; i++) v[i] = __float_as_uint(__uint_as_float(v[i]) + __uint_as_float(v2[i]));
        }
        const int col0 = nb * BN + c * 32;
        if (g.tma_store) {
          if (row_base >= g.M || col0 >= g.N) continue;  // warp-uniform: block fully outside C
          uint8_t* buf = stg + (e * C::STG + sbuf) * 4096;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(C::STG - 1) : "memory");
          __syncwarp();
          // ReLU'-gate operand: the 32 x 32 block of aux arrives by TMA into this warp's staging
          // buffer (coalesced, same swizzle as the store), instead of 32 per-row 128 B reads
          const bool aux_tma = g.splits == 1 && g.epi == GSG_EPI_MASK && g.aux_tma;
          if (aux_tma && lane == 0) {
            mbar_expect_tx(&auxbar[e], 4096);
            tma_load_2d(buf, &tmX, &auxbar[e], col0, row_base);
          }
          float x[32];
#pragma unroll
          for (int i = 0; i < 32; i++) x[i] = __uint_as_float(v[i]);
          if (g.splits == 1) {
            if (g.epi == GSG_EPI_RELU) {
#pragma unroll
              for (int i = 0; i < 32; i++) x[i] = fmaxf(x[i], 0.f);
              if (g.cbits) set_word(wb, c - c_begin, relu_bits(x, g.N - col0));
            } else if (aux_tma) {
              mbar_wait(&auxbar[e], aux_phase);
              aux_phase ^= 1;
#pragma unroll
              for (int j = 0; j < 8; j++) {
                const float4 m = *reinterpret_cast<const float4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4));
                x[4 * j] = m.x > 0.f ? x[4 * j] : 0.f;
                x[4 * j + 1] = m.y > 0.f ? x[4 * j + 1] : 0.f;
                x[4 * j + 2] = m.z > 0.f ? x[4 * j + 2] : 0.f;
                x[4 * j + 3] = m.w > 0.f ? x[4 * j + 3] : 0.f;
              }
            } else if (g.epi == GSG_EPI_MASK && row_ok && g.abits) {
              gate_bits(x, __ldg(g.abits + (int64_t)row * g.ldab + (col0 >> 5)));
            } else if (g.epi == GSG_EPI_MASK && row_ok) {
              const float* ax = g.aux + (int64_t)row * g.ldaux + col0;
              if (col0 + 32 <= g.N) {
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                  const float4 m = __ldg(reinterpret_cast<const float4*>(ax + i));
                  x[i] = m.x > 0.f ? x[i] : 0.f;
                  x[i + 1] = m.y > 0.f ? x[i + 1] : 0.f;
                  x[i + 2] = m.z > 0.f ? x[i + 2] : 0.f;
                  x[i + 3] = m.w > 0.f ? x[i + 3] : 0.f;
                }
              } else {
#pragma unroll
                for (int i = 0; i < 32; i++) if (col0 + i < g.N) x[i] = ax[i] > 0.f ? x[i] : 0.f;
              }
            }
            if (g.Clp && row_ok) {
              __nv_bfloat16* dl = g.Clp + (int64_t)row * g.ldclp + col0;
              if (col0 + 32 <= g.N) {
#pragma unroll
                for (int i = 0; i < 32; i += 8) {
                  __nv_bfloat162 p0 = __floats2bfloat162_rn(x[i], x[i + 1]);
                  __nv_bfloat162 p1 = __floats2bfloat162_rn(x[i + 2], x[i + 3]);
                  __nv_bfloat162 p2 = __floats2bfloat162_rn(x[i + 4], x[i + 5]);
                  __nv_bfloat162 p3 = __floats2bfloat162_rn(x[i + 6], x[i + 7]);
                  uint4 u;
                  u.x = *reinterpret_cast<uint32_t*>(&p0);
                  u.y = *reinterpret_cast<uint32_t*>(&p1);
                  u.z = *reinterpret_cast<uint32_t*>(&p2);
                  u.w = *reinterpret_cast<uint32_t*>(&p3);
                  *reinterpret_cast<uint4*>(dl + i) = u;
                }
              } else {
#pragma unroll
                for (int i = 0; i < 32; i++) if (col0 + i < g.N) dl[i] = __float2bfloat16_rn(x[i]);
              }
            }
          }
          // stage the 32 x 32 block (128B-swizzled rows) and store it with one TMA bulk-tensor op
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; j++)
            *reinterpret_cast<float4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            const int crow = g.splits > 1 ? s * g.mpad + row_base : row_base;
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                             reinterpret_cast<uint64_t>(&tmC)),
                         "r"(col0), "r"(crow), "r"(smem_u32(buf))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          if (++sbuf == C::STG) sbuf = 0;
          continue;
        }
        if (!row_ok || col0 >= g.N) continue;
        float x[32];
#pragma unroll
        for (int i = 0; i < 32; i++) x[i] = __uint_as_float(v[i]);
        if (g.splits > 1) {
          float* dst = g.ws + ((int64_t)s * g.mpad + row) * g.ldws + col0;
          if (col0 + 32 <= g.N) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(dst + i) = make_float4(x[i], x[i + 1], x[i + 2], x[i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; i++) if (col0 + i < g.N) dst[i] = x[i];
          }
          continue;
        }
        float* dst = g.C + (int64_t)row * g.ldc + col0;
        const bool full_chunk = col0 + 32 <= g.N;
        if (g.accumulate) {
          if (full_chunk) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 o = *reinterpret_cast<const float4*>(dst + i);
              x[i] += o.x; x[i + 1] += o.y; x[i + 2] += o.z; x[i + 3] += o.w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; i++) if (col0 + i < g.N) x[i] += dst[i];
          }
        }
        if (g.epi == GSG_EPI_RELU) {
#pragma unroll
          for (int i = 0; i < 32; i++) x[i] = fmaxf(x[i], 0.f);
          if (g.cbits) set_word(wb, c - c_begin, relu_bits(x, g.N - col0));
        } else if (g.epi == GSG_EPI_MASK && g.abits) {
          gate_bits(x, __ldg(g.abits + (int64_t)row * g.ldab + (col0 >> 5)));
        } else if (g.epi == GSG_EPI_MASK) {
          const float* ax = g.aux + (int64_t)row * g.ldaux + col0;
          if (full_chunk) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 m = __ldg(reinterpret_cast<const float4*>(ax + i));
              x[i] = m.x > 0.f ? x[i] : 0.f;
              x[i + 1] = m.y > 0.f ? x[i + 1] : 0.f;
              x[i + 2] = m.z > 0.f ? x[i + 2] : 0.f;
              x[i + 3] = m.w > 0.f ? x[i + 3] : 0.f;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; i++) if (col0 + i < g.N) x[i] = ax[i] > 0.f ? x[i] : 0.f;
          }
        }
        if (full_chunk) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(dst + i) = make_float4(x[i], x[i + 1], x[i + 2], x[i + 3]);
        } else {
#pragma unroll
          for (int i = 0; i < 32; i++) if (col0 + i < g.N) dst[i] = x[i];
        }
        if (g.Clp) {
          __nv_bfloat16* dl = g.Clp + (int64_t)row * g.ldclp + col0;
          if (full_chunk) {
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              __nv_bfloat162 p0 = __floats2bfloat162_rn(x[i], x[i + 1]);
              __nv_bfloat162 p1 = __floats2bfloat162_rn(x[i + 2], x[i + 3]);
              __nv_bfloat162 p2 = __floats2bfloat162_rn(x[i + 4], x[i + 5]);
              __nv_bfloat162 p3 = __floats2bfloat162_rn(x[i + 6], x[i + 7]);
              uint4 u;
              u.x = *reinterpret_cast<uint32_t*>(&p0);
              u.y = *reinterpret_cast<uint32_t*>(&p1);
              u.z = *reinterpret_cast<uint32_t*>(&p2);
              u.w = *reinterpret_cast<uint32_t*>(&p3);
              *reinterpret_cast<uint4*>(dl + i) = u;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; i++) if (col0 + i < g.N) dl[i] = __float2bfloat16_rn(x[i]);
          }
        }
      }
      if (g.cbits && row_ok) store_words<CPW>(g, row, nb * (BN / 32) + c_begin, wb);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (dual) {
          if constexpr (CTA2) {
            mbar_arrive_cluster(tempty_leader);
            mbar_arrive_cluster(tempty_leader + 8);
          } else {
            mbar_arrive(&tempty[0]);
            mbar_arrive(&tempty[1]);
          }
        } else {
          if constexpr (CTA2) mbar_arrive_cluster(tempty_leader + acc * 8);
          else mbar_arrive(&tempty[acc]);
        }
      }
      if (dual) acc_phase ^= 1;
      else if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (g.tma_store && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  if constexpr (CTA2) cluster_sync_all();
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CTA2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS)
                   : "memory");
  }
}

template <int BN, bool BF16, bool A_MN, bool B_MN, bool CTA2>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
           const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmX, const GemmArgs g) {
  gemm_body<BN, BF16, A_MN, B_MN, CTA2, false>(tmA, tmB, tmC, tmX, tmA, tmB, g);
}

template <int BN, bool BF16, bool A_MN, bool B_MN, bool CTA2>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_x3(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmX,
              const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2, const GemmArgs g) {
  gemm_body<BN, BF16, A_MN, B_MN, CTA2, true>(tmA, tmB, tmC, tmX, tmA2, tmB2, g);
}

// Epilogue of one reduced float4 (columns c .. c+3 of row; w = valid columns).
// With a ReLU bitmask output (FP32X3 splits only) the 4 columns' bits are OR-ed into their word,
// which the GEMM's tile epilogue zeroed (OR commutes: the result does not depend on the order).
__device__ __forceinline__ void reduce_store4(const GemmArgs& g, int row, int c, int w, const float (&x)[4]) {
  float* dst = g.C + (int64_t)row * g.ldc + c;
  uint32_t nib = 0;
  for (int j = 0; j < w; j++) {
    float y = x[j];
    if (g.accumulate) y += dst[j];
    if (g.epi == GSG_EPI_RELU) y = fmaxf(y, 0.f);
    else if (g.epi == GSG_EPI_MASK && g.abits) y = (g.abits[(int64_t)row * g.ldab + ((c + j) >> 5)] >> ((c + j) & 31)) & 1u ? y : 0.f;
    else if (g.epi == GSG_EPI_MASK) y = g.aux[(int64_t)row * g.ldaux + c + j] > 0.f ? y : 0.f;
    dst[j] = y;
    if (g.Clp) g.Clp[(int64_t)row * g.ldclp + c + j] = __float2bfloat16_rn(y);
    nib |= (y > 0.f ? 1u : 0u) << j;
  }
  if (g.cbits && nib) atomicOr(g.cbits + (int64_t)row * g.ldcb + (c >> 5), nib << (c & 31));
}

// C = epi(sum_s ws[s]) in a fixed split order (deterministic split-K reduction), one thread per
// output float4 (few splits, many outputs).
__global__ void k_splitk_reduce(GemmArgs g) {
  const int n4 = (g.N + 3) / 4;
  const int64_t total = (int64_t)g.M * n4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(i / n4);
    const int c = (int)(i % n4) * 4;
    float x[4] = {0.f, 0.f, 0.f, 0.f};
    // ws rows are padded to ldws (multiple of 8 >= N): float4 loads never leave the row. Loads
    // are issued 8 at a time (independent), sums applied in split order (deterministic).
    const float4* p = reinterpret_cast<const float4*>(g.ws + (int64_t)row * g.ldws + c);
    const int64_t sstride4 = (int64_t)g.mpad * g.ldws / 4;
    int s = 0;
    for (; s + 8 <= g.splits; s += 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) v[u] = __ldg(p + (s + u) * sstride4);
#pragma unroll
      for (int u = 0; u < 8; u++) { x[0] += v[u].x; x[1] += v[u].y; x[2] += v[u].z; x[3] += v[u].w; }
    }
    if (s < g.splits) {  // remaining < 8 splits: predicated loads, all in flight together
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) v[u] = s + u < g.splits ? __ldg(p + (s + u) * sstride4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (s + u < g.splits) { x[0] += v[u].x; x[1] += v[u].y; x[2] += v[u].z; x[3] += v[u].w; }
    }
    reduce_store4(g, row, c, min(4, g.N - c), x);
  }
}

// Same reduction, one warp per output float4 (many splits, few outputs: e.g. a 1024 x 41 head
// gradient over K = n cut into 64 pieces): lane l sums splits l, l + 32, ... in order, then a
// fixed xor-butterfly combines the lanes (deterministic; a different but fixed association).
__global__ void k_splitk_reduce_warp(GemmArgs g) {
  const int n4 = (g.N + 3) / 4;
  const int64_t total = (int64_t)g.M * n4;
  const int lane = threadIdx.x & 31;
  const int64_t W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t sstride4 = (int64_t)g.mpad * g.ldws / 4;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < total; i += W) {
    const int row = (int)(i / n4);
    const int c = (int)(i % n4) * 4;
    const float4* p = reinterpret_cast<const float4*>(g.ws + (int64_t)row * g.ldws + c);
    float x[4] = {0.f, 0.f, 0.f, 0.f};
    for (int s = lane; s < g.splits; s += 32) {
      const float4 v = __ldg(p + s * sstride4);
      x[0] += v.x; x[1] += v.y; x[2] += v.z; x[3] += v.w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int j = 0; j < 4; j++) x[j] += __shfl_xor_sync(0xffffffffu, x[j], o);
    if (lane == 0) reduce_store4(g, row, c, min(4, g.N - c), x);
  }
}

// K = 0: C = epi(0) (+ C when accumulating)
__global__ void k_fill_epi(GemmArgs g) {
  const int64_t total = (int64_t)g.M * g.N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(i / g.N), c = (int)(i % g.N);
    float y = g.accumulate ? g.C[(int64_t)row * g.ldc + c] : 0.f;
    if (g.epi == GSG_EPI_RELU) y = fmaxf(y, 0.f);
    else if (g.epi == GSG_EPI_MASK) y = 0.f;  // accumulate is NONE-only: y is 0 here
    g.C[(int64_t)row * g.ldc + c] = y;
    if (g.Clp) g.Clp[(int64_t)row * g.ldclp + c] = __float2bfloat16_rn(y);
  }
}

__global__ void k_to_bf16(int rows, int cols, const float* __restrict__ src, int64_t lds, __nv_bfloat16* __restrict__ dst,
                          int64_t ldd) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / cols), c = (int)(i % cols);
    dst[(int64_t)r * ldd + c] = __float2bfloat16_rn(src[(int64_t)r * lds + c]);
  }
}

// 4 columns per thread (float4 in, 4 x bf16 = 8 bytes out): cols, lds, ldd multiples of 4.
__global__ void k_to_bf16_v4(int rows, int cols4, const float4* __restrict__ src, int64_t lds4, uint2* __restrict__ dst,
                             int64_t ldd4) {
  const int64_t total = (int64_t)rows * cols4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / cols4), c = (int)(i % cols4);
    const float4 v = __ldg(src + (int64_t)r * lds4 + c);
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 p;
    p.x = *reinterpret_cast<uint32_t*>(&lo);
    p.y = *reinterpret_cast<uint32_t*>(&hi);
    dst[(int64_t)r * ldd4 + c] = p;
  }
}

// GSG_PREC_FP32X3 operand split: x = hi + lo, hi = tf32 round-to-nearest of x (an fp32 with the
// low 13 mantissa bits zero, read exactly by kind::tf32), lo = x - hi (exact in fp32). The three
// copies c0, c1, c2 (each hi or lo per `pat`, bit j = 1 -> copy j is lo) are stacked along K:
// along the columns of a K-major operand (dst row r = [c0 | c1 | c2], K columns each) or along
// the rows of an MN-major one (dst rows [c0 ; c1 ; c2], K rows each).
__global__ void k_split3(int rows, int cols, const float* __restrict__ src, int64_t lds, float* __restrict__ dst,
                         int64_t ldd, int along_cols, int K, int pat) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / cols), c = (int)(i % cols);
    const float x = src[(int64_t)r * lds + c];
    uint32_t hb;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(x));
    const float hi = __uint_as_float(hb), lo = x - hi;
#pragma unroll
    for (int j = 0; j < 3; j++) {
      const float v = (pat >> j) & 1 ? lo : hi;
      if (along_cols) dst[(int64_t)r * ldd + (int64_t)j * K + c] = v;
      else dst[((int64_t)j * K + r) * ldd + c] = v;
    }
  }
}

// FP32X3 with implicit hi: kind::tf32 reads an fp32 operand by truncating it to tf32 (measured:
// 1 + 0.75 ulp_tf32 enters as 1), so the unmodified operand IS hi = trunc_tf32(x) to the tensor
// core and only lo = x - trunc_tf32(x) (exact in fp32) is materialized, in the operand's own
// stored shape. One warp per row, lanes along the row.
// raw != nullptr: also copy x itself there (same ldd), for an operand whose stride or alignment
// TMA cannot read directly.
__global__ void k_split_lo(int rows, int cols, const float* __restrict__ src, int64_t lds, float* __restrict__ dst,
                           int64_t ldd, float* __restrict__ raw) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += warps) {
    const float* s = src + (int64_t)r * lds;
    float* d = dst + (int64_t)r * ldd;
    if ((cols & 3) == 0 && (lds & 3) == 0 && ((uintptr_t)src & 15) == 0) {  // ldd % 4 == 0, dst aligned
      const int n4 = cols / 4;
      for (int c0 = lane; c0 < n4; c0 += 128) {  // 4 loads in flight per lane
        float4 x[4];
#pragma unroll
        for (int u = 0; u < 4; u++)
          x[u] = c0 + 32 * u < n4 ? __ldg(reinterpret_cast<const float4*>(s) + c0 + 32 * u) : make_float4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int c = c0 + 32 * u;
          if (c >= n4) break;
          float4 y;
          y.x = x[u].x - __uint_as_float(__float_as_uint(x[u].x) & 0xFFFFE000u);
          y.y = x[u].y - __uint_as_float(__float_as_uint(x[u].y) & 0xFFFFE000u);
          y.z = x[u].z - __uint_as_float(__float_as_uint(x[u].z) & 0xFFFFE000u);
          y.w = x[u].w - __uint_as_float(__float_as_uint(x[u].w) & 0xFFFFE000u);
          reinterpret_cast<float4*>(d)[c] = y;
          if (raw) reinterpret_cast<float4*>(raw + (int64_t)r * ldd)[c] = x[u];
        }
      }
    } else {
      for (int c = lane; c < cols; c += 32) {
        const float x = __ldg(s + c);
        d[c] = x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
        if (raw) raw[(int64_t)r * ldd + c] = x;
      }
    }
  }
}

// --------------------------------------------------------------------------- host helpers
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int get_encode() {
  static std::once_flag once;
  static int rc = GSG_OK;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) {
      rc = fail(GSG_ECUDA, "cuTensorMapEncodeTiled unavailable");
      return;
    }
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return rc;
}

// 2-D row-major tensor [rows x cols] (ld elements), box {box_cols, box_rows}, 128B swizzle.
int make_map(CUtensorMap* m, const void* base, bool bf16, int64_t rows, int64_t cols, int64_t ld, int box_cols,
             int box_rows, bool mn_major) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * (bf16 ? 2 : 4))};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                        const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        (mn_major && !bf16) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(GSG_EINVAL, "cuTensorMapEncodeTiled failed (%d): rows=%lld cols=%lld ld=%lld box=%dx%d", (int)r,
                (long long)rows, (long long)cols, (long long)ld, box_cols, box_rows);
  return GSG_OK;
}

// fp32 [rows x cols] store map, box 32 x 32, 128B swizzle (matches the epilogue staging layout)
int make_store_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(GSG_EINVAL, "cuTensorMapEncodeTiled(store) failed (%d): rows=%lld cols=%lld ld=%lld", (int)r,
                (long long)rows, (long long)cols, (long long)ld);
  return GSG_OK;
}

template <int BN, bool BF16, bool A_MN, bool B_MN, bool CTA2>
int run_gemm(gsg_ctx* ctx, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, const CUtensorMap& mx,
             const CUtensorMap& ma2, const CUtensorMap& mb2, const GemmArgs& g) {
  using C = Cfg<BN, BF16, CTA2>;
  auto kern = k_gemm<BN, BF16, A_MN, B_MN, CTA2>;
  // function attributes are per device: set once for each device a context uses (racing
  // threads may both set them, which is harmless)
  static std::atomic<uint64_t> attr_devs{0};
  const uint64_t dbit = 1ull << (ctx->device & 63);
  if (!(attr_devs.load(std::memory_order_acquire) & dbit)) {
    GSG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    if (CTA2) GSG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
    if constexpr (!BF16) {
      auto kern3 = k_gemm_x3<BN, false, A_MN, B_MN, CTA2>;
      GSG_CUDA(cudaFuncSetAttribute(kern3, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
      if (CTA2) GSG_CUDA(cudaFuncSetAttribute(kern3, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
    }
    attr_devs.fetch_or(dbit, std::memory_order_release);
  }
  const int tiles = g.num_m * g.num_n * g.splits;
  int grid;
  if (CTA2) {
    const int pairs = ctx->num_sms / 2;
    grid = 2 * (tiles < pairs ? tiles : pairs);
  } else {
    grid = tiles < ctx->num_sms ? tiles : ctx->num_sms;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CTA2 ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if constexpr (!BF16) {
    if (g.x3nkb) GSG_CUDA(cudaLaunchKernelEx(&cfg, k_gemm_x3<BN, false, A_MN, B_MN, CTA2>, ma, mb, mc, mx, ma2, mb2, g));
    else GSG_CUDA(cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, mx, g));
  } else {
    GSG_CUDA(cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, mx, g));
  }
  count_launch(ctx);
  return GSG_OK;
}

template <int BN, bool BF16, bool CTA2>
int dispatch_major(gsg_ctx* ctx, bool a_mn, bool b_mn, const CUtensorMap& ma, const CUtensorMap& mb,
                   const CUtensorMap& mc, const CUtensorMap& mx, const CUtensorMap& ma2, const CUtensorMap& mb2,
                   const GemmArgs& g) {
  if (!a_mn && !b_mn) return run_gemm<BN, BF16, false, false, CTA2>(ctx, ma, mb, mc, mx, ma2, mb2, g);
  if (!a_mn && b_mn) return run_gemm<BN, BF16, false, true, CTA2>(ctx, ma, mb, mc, mx, ma2, mb2, g);
  if (a_mn && !b_mn) return run_gemm<BN, BF16, true, false, CTA2>(ctx, ma, mb, mc, mx, ma2, mb2, g);
  return run_gemm<BN, BF16, true, true, CTA2>(ctx, ma, mb, mc, mx, ma2, mb2, g);
}

}  // namespace

namespace {
int gemm_launch_impl(gsg_ctx* ctx, int M, int N, int K, const void* A, int64_t lda, int transA, const void* B,
                     int64_t ldb, int transB, float* Cp, int64_t ldc, void* Clp, int64_t ldclp, int precision,
                     int epilogue, const float* aux, int64_t ldaux, int split_k, int accumulate, const BitsIO& bits,
                     bool x3, const float* Alo = nullptr, int64_t ldalo = 0, const float* Blo = nullptr,
                     int64_t ldblo = 0);
}  // namespace

int gemm_launch(gsg_ctx* ctx, int M, int N, int K, const void* A, int64_t lda, int transA, const void* B, int64_t ldb,
                int transB, float* Cp, int64_t ldc, void* Clp, int64_t ldclp, int precision, int epilogue,
                const float* aux, int64_t ldaux, int split_k, int accumulate, const BitsIO& bits, const X3Lo& pre) {
  const bool x3 = precision == GSG_PREC_FP32X3;  // precomputed lo operands mean nothing otherwise
  return gemm_launch_impl(ctx, M, N, K, A, lda, transA, B, ldb, transB, Cp, ldc, Clp, ldclp, precision, epilogue, aux,
                          ldaux, split_k, accumulate, bits, false, x3 ? pre.a : nullptr, pre.lda, x3 ? pre.b : nullptr,
                          pre.ldb);
}

static int split_grid(gsg_ctx* ctx, int64_t rows) {
  return (int)std::min<int64_t>(std::max<int64_t>((rows * 32 + 255) / 256, 1), (int64_t)ctx->num_sms * 8);
}

int split_lo_launch(gsg_ctx* ctx, int rows, int cols, const float* src, int64_t lds, float* dst, int64_t ldd) {
  GSG_CHECK(rows >= 0 && cols >= 0 && lds >= cols && ldd >= cols && ldd % 4 == 0 && (uintptr_t)dst % 16 == 0,
            GSG_EINVAL, "split_lo: bad shape");
  if (rows == 0 || cols == 0) return GSG_OK;
  k_split_lo<<<split_grid(ctx, rows), 256, 0, ctx->stream>>>(rows, cols, src, lds, dst, ldd, nullptr);
  count_launch(ctx);
  GSG_CUDA(cudaGetLastError());
  return GSG_OK;
}

bool x3_implicit() {
  static const int v = getenv("GSG_X3_IMPLICIT") ? atoi(getenv("GSG_X3_IMPLICIT")) : 1;  // A/B
  return v != 0;
}

namespace {
int gemm_launch_impl(gsg_ctx* ctx, int M, int N, int K, const void* A, int64_t lda, int transA, const void* B,
                     int64_t ldb, int transB, float* Cp, int64_t ldc, void* Clp, int64_t ldclp, int precision,
                     int epilogue, const float* aux, int64_t ldaux, int split_k, int accumulate, const BitsIO& bits,
                     bool x3, const float* Alo, int64_t ldalo, const float* Blo, int64_t ldblo) {
  GSG_CHECK(precision == GSG_PREC_TF32 || precision == GSG_PREC_BF16 || precision == GSG_PREC_FP32X3, GSG_EINVAL,
            "bad precision %d", precision);
  GSG_CHECK(epilogue >= GSG_EPI_NONE && epilogue <= GSG_EPI_MASK, GSG_EINVAL, "bad epilogue %d", epilogue);
  GSG_CHECK(M >= 0 && N >= 0 && K >= 0, GSG_EINVAL, "negative GEMM dims");
  GSG_CHECK(!accumulate || epilogue == GSG_EPI_NONE, GSG_EINVAL, "accumulate only with GSG_EPI_NONE");
  if (M == 0 || N == 0) return GSG_OK;  // nothing to write: no pointer is read
  GSG_CHECK(Cp && ldc >= N && ldc % 4 == 0 && (uintptr_t)Cp % 16 == 0, GSG_EINVAL,
            "C: need ldc >= N, ldc %% 4 == 0, 16B alignment (ldc=%lld N=%d)", (long long)ldc, N);
  GSG_CHECK(!Clp || (ldclp >= N && ldclp % 8 == 0 && (uintptr_t)Clp % 16 == 0), GSG_EINVAL,
            "Clp: need ldclp >= N, ldclp %% 8 == 0, 16B alignment");
  const int64_t nwords = (N + 31) / 32;
  GSG_CHECK(epilogue != GSG_EPI_MASK || bits.in ||
                (aux && ldaux >= N && ldaux % 4 == 0 && (uintptr_t)aux % 16 == 0),
            GSG_EINVAL, "EPI_MASK needs aux with ldaux >= N, ldaux %% 4 == 0, 16B alignment (or a bitmask gate)");
  GSG_CHECK(!bits.in || (epilogue == GSG_EPI_MASK && bits.ldi >= nwords && (uintptr_t)bits.in % 4 == 0), GSG_EINVAL,
            "bitmask gate needs GSG_EPI_MASK and ldauxb >= ceil(N/32) (ldauxb=%lld)", (long long)bits.ldi);
  GSG_CHECK(!bits.out || (epilogue == GSG_EPI_RELU && bits.ldo >= nwords && (uintptr_t)bits.out % 4 == 0), GSG_EINVAL,
            "bitmask output needs GSG_EPI_RELU and ldcb >= ceil(N/32) (ldcb=%lld)", (long long)bits.ldo);
  if (precision == GSG_PREC_FP32X3 && K > 0 && x3_implicit()) {
    // 3xTF32 with implicit hi: one TF32 GEMM over K' = 3K, segments [A | A | Alo] x [B ; Blo ; B]
    // (the tensor core truncates the fp32 operand to hi itself); only Alo and Blo are written
    GSG_CHECK(A && B, GSG_EINVAL, "A and B must be non-NULL");
    const int64_t ar = transA ? K : M, ac = transA ? M : K, br = transB ? N : K, bc = transB ? K : N;
    GSG_CHECK(lda >= ac && ldb >= bc, GSG_EINVAL, "lda / ldb below the stored widths");
    const int64_t ldal = (ac + 3) / 4 * 4, ldbl = (bc + 3) / 4 * 4;
    // an operand TMA cannot read in place (row pitch or base not 16-byte aligned) is copied too
    const bool copy_a = lda % 4 != 0 || (uintptr_t)A % 16 != 0, copy_b = ldb % 4 != 0 || (uintptr_t)B % 16 != 0;
    DevBuf* ws = ctx->side_ws ? ctx->ws_x3_side : ctx->ws_x3;
    if (!(Alo && !copy_a))
      if (int rc = ws[0].reserve(sizeof(float) * ar * ldal * (copy_a ? 2 : 1))) return rc;
    if (!(Blo && !copy_b))
      if (int rc = ws[1].reserve(sizeof(float) * br * ldbl * (copy_b ? 2 : 1))) return rc;
    float* Al = static_cast<float*>(ws[0].ptr);
    float* Bl = static_cast<float*>(ws[1].ptr);
    float* Ar = copy_a ? Al + ar * ldal : nullptr;
    float* Br = copy_b ? Bl + br * ldbl : nullptr;
    // a lo the caller computed (Alo / Blo here, X3Lo) is used as is for an operand TMA reads in place
    const bool pre_a = Alo && !copy_a, pre_b = Blo && !copy_b;
    if (!pre_a)
      k_split_lo<<<split_grid(ctx, ar), 256, 0, ctx->stream>>>((int)ar, (int)ac, static_cast<const float*>(A), lda, Al,
                                                             ldal, Ar);
    if (!pre_b)
      k_split_lo<<<split_grid(ctx, br), 256, 0, ctx->stream>>>((int)br, (int)bc, static_cast<const float*>(B), ldb, Bl,
                                                             ldbl, Br);
    count_launch(ctx, (pre_a ? 0 : 1) + (pre_b ? 0 : 1));
    GSG_CUDA(cudaGetLastError());
    return gemm_launch_impl(ctx, M, N, K, copy_a ? Ar : A, copy_a ? ldal : lda, transA, copy_b ? Br : B,
                            copy_b ? ldbl : ldb, transB, Cp, ldc, Clp, ldclp, GSG_PREC_TF32, epilogue, aux, ldaux,
                            split_k, accumulate, bits, true, pre_a ? Alo : Al, pre_a ? ldalo : ldal, pre_b ? Blo : Bl,
                            pre_b ? ldblo : ldbl);
  }
  if (precision == GSG_PREC_FP32X3 && K > 0) {
    // 3xTF32 (GSG_X3_IMPLICIT=0): one TF32 GEMM over K' = 3K on split copies [Ahi | Ahi | Alo] x
    // [Bhi ; Blo ; Bhi], hi rounded to nearest
    GSG_CHECK(A && B, GSG_EINVAL, "A and B must be non-NULL");
    GSG_CHECK(3LL * K < (int64_t)INT32_MAX, GSG_EUNSUPPORTED, "FP32X3 needs 3K < 2^31 (K=%d)", K);
    const int64_t K3 = 3LL * K;
    // stored shapes: A is (transA ? K x M : M x K), B is (transB ? N x K : K x N)
    const int64_t ar = transA ? K : M, ac = transA ? M : K, br = transB ? N : K, bc = transB ? K : N;
    GSG_CHECK(lda >= ac && ldb >= bc, GSG_EINVAL, "lda / ldb below the stored widths");
    const int64_t lda3 = transA ? (M + 3) / 4 * 4 : (K3 + 3) / 4 * 4;  // K-major: K' along columns
    const int64_t ldb3 = transB ? (K3 + 3) / 4 * 4 : (N + 3) / 4 * 4;
    const int64_t a3 = transA ? K3 * lda3 : (int64_t)M * lda3, b3 = transB ? (int64_t)N * ldb3 : K3 * ldb3;
    DevBuf* ws = ctx->side_ws ? ctx->ws_x3_side : ctx->ws_x3;
    if (int rc = ws[0].reserve(sizeof(float) * a3)) return rc;
    if (int rc = ws[1].reserve(sizeof(float) * b3)) return rc;
    float* A3 = static_cast<float*>(ws[0].ptr);
    float* B3 = static_cast<float*>(ws[1].ptr);
    auto grid_for = [&](int64_t n) {
      int64_t gd = (n + 255) / 256;
      return (int)std::min<int64_t>(std::max<int64_t>(gd, 1), (int64_t)ctx->num_sms * 8);
    };
    // A: hi, hi, lo (pattern 0b100); B: hi, lo, hi (0b010)
    k_split3<<<grid_for(ar * ac), 256, 0, ctx->stream>>>((int)ar, (int)ac, static_cast<const float*>(A), lda, A3, lda3,
                                                        transA ? 0 : 1, K, 4);
    k_split3<<<grid_for(br * bc), 256, 0, ctx->stream>>>((int)br, (int)bc, static_cast<const float*>(B), ldb, B3, ldb3,
                                                        transB ? 1 : 0, K, 2);
    count_launch(ctx, 2);
    GSG_CUDA(cudaGetLastError());
    return gemm_launch_impl(ctx, M, N, (int)K3, A3, lda3, transA, B3, ldb3, transB, Cp, ldc, Clp, ldclp,
                            GSG_PREC_TF32, epilogue, aux, ldaux, split_k, accumulate, bits, true);
  }
  if (precision == GSG_PREC_FP32X3) precision = GSG_PREC_TF32;  // K = 0: the epilogue of zero
  const bool bf16 = precision == GSG_PREC_BF16;
  const double kx = Alo ? 3.0 : 1.0;  // implicit-hi FP32X3 executes K' = 3K
  ProfScope ps(ctx, GSG_K_GEMM,
               (double)(bf16 ? 2 : 4) * kx * ((double)M * K + (double)K * N) + 4.0 * M * N, 2.0 * M * N * K * kx);
  const int elem = bf16 ? 2 : 4;
  GemmArgs g{};
  g.M = M; g.N = N; g.K = K;
  g.C = Cp; g.ldc = ldc;
  g.Clp = reinterpret_cast<__nv_bfloat16*>(Clp); g.ldclp = ldclp;
  g.aux = bits.in ? nullptr : aux; g.ldaux = ldaux; g.epi = epilogue; g.accumulate = accumulate;
  g.abits = bits.in; g.ldab = bits.ldi;
  g.cbits = bits.out; g.ldcb = bits.ldo;
  if (K == 0) {
    if (bits.out) GSG_CUDA(cudaMemset2DAsync(bits.out, bits.ldo * 4, 0, nwords * 4, M, ctx->stream));  // ReLU(0) = 0
    k_fill_epi<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(g);
    count_launch(ctx);
    GSG_CUDA(cudaGetLastError());
    return GSG_OK;
  }
  GSG_CHECK(A && B, GSG_EINVAL, "A and B must be non-NULL");
  // stored shapes: A is (transA ? K x M : M x K), B is (transB ? N x K : K x N)
  const int64_t a_cols = transA ? M : K, b_cols = transB ? K : N;
  GSG_CHECK(lda >= a_cols && (lda * elem) % 16 == 0 && (uintptr_t)A % 16 == 0, GSG_EINVAL,
            "A: lda=%lld must be >= %lld with 16-byte rows/alignment", (long long)lda, (long long)a_cols);
  GSG_CHECK(ldb >= b_cols && (ldb * elem) % 16 == 0 && (uintptr_t)B % 16 == 0, GSG_EINVAL,
            "B: ldb=%lld must be >= %lld with 16-byte rows/alignment", (long long)ldb, (long long)b_cols);
  int rc = get_encode();
  if (rc) return rc;
  const int BN = N <= 128 ? 128 : 256;
  // pair (cta_group::2, 256-row tiles) whenever the shape fills the pair tile; GSG_GEMM_1CTA=1 forces 1-CTA.
  // (128-wide pair tiles would cut the last-wave waste on 20000 x 1024 but measured 1.35x slower.)
  static const bool force1 = getenv("GSG_GEMM_1CTA") && atoi(getenv("GSG_GEMM_1CTA")) == 1;
  const bool cta2 = !force1 && BN == 256 && M > BM;
  const int BMT = cta2 ? 2 * BM : BM;
  const int BK = 128 / elem, mnrow = 128 / elem;
  g.num_m = (M + BMT - 1) / BMT;
  g.num_n = (N + BN - 1) / BN;
  g.num_kb = (K + BK - 1) / BK;
  if (Alo) {  // K' = 3 segments of num_kb k-blocks each
    g.x3nkb = g.num_kb;
    g.num_kb *= 3;
  }
  const int base_tiles = g.num_m * g.num_n;
  int splits = split_k;
  if (splits <= 0) {
    // Pick the K split that minimizes modeled time: waves x (k-blocks per split + epilogue
    // overhead of ~2 k-blocks) + the fixed-order reduction (reads s partials, writes C).
    const int units = cta2 ? ctx->num_sms / 2 : ctx->num_sms;
    const double t_kb_us = cta2 ? 0.52 : 0.55;                 // one k-block of one tile (TF32)
    const double red_us_per_split = (double)M * N * 4.0 / 5.0e6;  // ~5 TB/s streaming
    int max_s = g.num_kb / 4;                                   // keep >= 4 k-blocks per split
    if (max_s > 64) max_s = 64;
    if (max_s < 1) max_s = 1;
    if (base_tiles * 2 > units) max_s = 1;  // the grid is already at least half full: no split
                                            // (measured: the reduction costs more than the tail)
    // a narrow forkable GEMM (the head's dW_mlp, which runs on the side stream beside dH_L)
    // takes at most 12 K pieces: fewer SMs taken from the critical-path GEMM and a cheaper
    // reduction (config 5 2.954 -> 2.948 ms, config 3 0.594 -> 0.590 ms;
    // profiles/r01_gemm_side_split_cap_ab.txt). The cap applies to every forkable GEMM, forked
    // or serialized (GSG_BWD_FORK=0, profiling), so both pick the same split and workspace: a
    // serialized pass captured into a CUDA graph never has to grow the workspace.
    if (ctx->side_ws && N <= 128 && max_s > 12) max_s = 12;
    double best = 1e30;
    splits = 1;
    for (int s = 1; s <= max_s; s++) {
      const int kbps = (g.num_kb + s - 1) / s;
      const int waves = (base_tiles * s + units - 1) / units;
      const double t = waves * (kbps + 2) * t_kb_us + (s > 1 ? (s + 1) * red_us_per_split : 0.0);
      if (t < best * 0.97) { best = t; splits = s; }
    }
  }
  // GSG_PREC_FP32X3 (K here is the tripled K'): at most 32 k-blocks (K' = 1024) per automatic
  // split -- the fp32 sum inside one tensor-core accumulator drifts with the piece length
  // (max-normalized 1.5e-5 at K' = 3600, 4.9e-5 at 12000, measured), past the 1e-5 the split
  // precision is for; the pieces are summed by the fixed-order reduction in fp32, which also
  // writes the ReLU bitmask then
  // (the implicit-hi kernel accumulates each split in two TMEM halves: 64 k-blocks per split)
  const int x3_cap = Alo ? 64 : 32;
  if (split_k <= 0 && x3 && splits < (g.num_kb + x3_cap - 1) / x3_cap) splits = (g.num_kb + x3_cap - 1) / x3_cap;
  // TF32 / BF16: the bitmask is written by the tile epilogue, not the split-K reduction
  if (bits.out && !x3) splits = 1;
  if (splits > g.num_kb) splits = g.num_kb;
  g.kb_per_split = (g.num_kb + splits - 1) / splits;
  // two TMEM halves per tile only where a piece is longer than the 32-k-block drift bound; shorter
  // pieces keep the accumulator ping-pong (epilogue of one tile under the next tile's mainloop)
  g.x3dual = Alo && g.kb_per_split > 32 ? 1 : 0;
  g.splits = (g.num_kb + g.kb_per_split - 1) / g.kb_per_split;  // no empty split
  g.mpad = g.num_m * BMT;
  if (g.splits > 1) {
    g.ldws = (N + 7) / 8 * 8;
    // a GEMM forked onto the side stream may run concurrently with one on the context stream:
    // the forkable GEMMs (dW, dW_mlp) always use their own workspace, forked or not, so that a
    // serialized (profiling) pass inside a graph capture never has to grow it
    DevBuf& wsk = ctx->side_ws ? ctx->ws_splitk_side : ctx->ws_splitk;
    rc = wsk.reserve((size_t)g.splits * g.mpad * g.ldws * sizeof(float));
    if (rc) return rc;
    g.ws = static_cast<float*>(wsk.ptr);
  }
  // instruction descriptor: D=F32, A/B = TF32 (2) or BF16 (1), majorness, N>>3, M>>4
  const uint32_t fmt = bf16 ? 1u : 2u;
  g.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(transA ? 1 : 0) << 15) |
            ((uint32_t)(transB ? 0 : 1) << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BMT >> 4) << 24);
  const int BNC = cta2 ? BN / 2 : BN;  // B rows staged per CTA
  CUtensorMap ma, mb;
  if (transA) rc = make_map(&ma, A, bf16, K, M, lda, mnrow, BK, true);   // MN-major A (stored K x M)
  else rc = make_map(&ma, A, bf16, M, K, lda, BK, BM, false);            // K-major A (stored M x K)
  if (rc) return rc;
  if (transB) rc = make_map(&mb, B, bf16, N, K, ldb, BK, BNC, false);    // K-major B (stored N x K)
  else rc = make_map(&mb, B, bf16, K, N, ldb, mnrow, BK, true);          // MN-major B (stored K x N)
  if (rc) return rc;
  CUtensorMap ma2 = ma, mb2 = mb;  // the lo operands of an implicit-hi FP32X3 GEMM (same boxes)
  if (Alo) {
    if (transA) rc = make_map(&ma2, Alo, false, K, M, ldalo, mnrow, BK, true);
    else rc = make_map(&ma2, Alo, false, M, K, ldalo, BK, BM, false);
    if (rc) return rc;
    if (transB) rc = make_map(&mb2, Blo, false, N, K, ldblo, BK, BNC, false);
    else rc = make_map(&mb2, Blo, false, K, N, ldblo, mnrow, BK, true);
    if (rc) return rc;
  }
  // epilogue store map: C itself, or the split-K workspace [splits * mpad x ldws]
  CUtensorMap mc;
  g.tma_store = accumulate ? 0 : 1;
  if (g.splits > 1) rc = make_store_map(&mc, g.ws, (int64_t)g.splits * g.mpad, N, g.ldws);
  else rc = make_store_map(&mc, Cp, M, N, ldc);
  if (rc) return rc;
  // gate operand map (same 32 x 32 swizzled box as the store) for GSG_EPI_MASK
  CUtensorMap mx = mc;
  g.aux_tma = 0;
  if (epilogue == GSG_EPI_MASK && !bits.in && g.tma_store && g.splits == 1) {
    if ((rc = make_store_map(&mx, aux, M, N, ldaux))) return rc;
    g.aux_tma = 1;
  }
  const bool a_mn = transA, b_mn = !transB;
  if (cta2) {
    rc = bf16 ? dispatch_major<256, true, true>(ctx, a_mn, b_mn, ma, mb, mc, mx, ma2, mb2, g)
              : dispatch_major<256, false, true>(ctx, a_mn, b_mn, ma, mb, mc, mx, ma2, mb2, g);
  } else if (bf16) {
    rc = BN == 128 ? dispatch_major<128, true, false>(ctx, a_mn, b_mn, ma, mb, mc, mx, ma2, mb2, g)
                   : dispatch_major<256, true, false>(ctx, a_mn, b_mn, ma, mb, mc, mx, ma2, mb2, g);
  } else {
    rc = BN == 128 ? dispatch_major<128, false, false>(ctx, a_mn, b_mn, ma, mb, mc, mx, ma2, mb2, g)
                   : dispatch_major<256, false, false>(ctx, a_mn, b_mn, ma, mb, mc, mx, ma2, mb2, g);
  }
  if (rc) return rc;
  if (g.splits > 1) {
    const int64_t total = (int64_t)M * ((N + 3) / 4);
    if (g.splits >= 16 && total < (int64_t)ctx->num_sms * 256) {
      int64_t grid = (total * 32 + 255) / 256;  // one warp per output float4
      if (grid > ctx->num_sms * 8) grid = ctx->num_sms * 8;
      k_splitk_reduce_warp<<<(int)grid, 256, 0, ctx->stream>>>(g);
    } else {
      int grid = (int)((total + 255) / 256);
      if (grid > ctx->num_sms * 8) grid = ctx->num_sms * 8;
      k_splitk_reduce<<<grid, 256, 0, ctx->stream>>>(g);
    }
    count_launch(ctx);
    GSG_CUDA(cudaGetLastError());
  }
  return GSG_OK;
}

}  // namespace

int to_bf16_launch(gsg_ctx* ctx, int rows, int cols, const float* src, int64_t lds, void* dst, int64_t ldd) {
  GSG_CHECK(rows >= 0 && cols >= 0 && lds >= cols && ldd >= cols, GSG_EINVAL, "bad to_bf16 shape");
  if (rows == 0 || cols == 0) return GSG_OK;
  ProfScope ps(ctx, GSG_K_OTHER, 6.0 * rows * cols, 0.0);
  if (cols % 4 == 0 && lds % 4 == 0 && ldd % 4 == 0 && (uintptr_t)src % 16 == 0 && (uintptr_t)dst % 8 == 0) {
    const int64_t total = (int64_t)rows * (cols / 4);
    int grid = (int)((total + 255) / 256);
    if (grid > ctx->num_sms * 8) grid = ctx->num_sms * 8;
    k_to_bf16_v4<<<grid, 256, 0, ctx->stream>>>(rows, cols / 4, reinterpret_cast<const float4*>(src), lds / 4,
                                                static_cast<uint2*>(dst), ldd / 4);
    count_launch(ctx);
    GSG_CUDA(cudaGetLastError());
    return GSG_OK;
  }
  int64_t total = (int64_t)rows * cols;
  int grid = (int)((total + 255) / 256);
  if (grid > ctx->num_sms * 8) grid = ctx->num_sms * 8;
  k_to_bf16<<<grid, 256, 0, ctx->stream>>>(rows, cols, src, lds, static_cast<__nv_bfloat16*>(dst), ldd);
  count_launch(ctx);
  GSG_CUDA(cudaGetLastError());
  return GSG_OK;
}

}  // namespace gsg
