// sampler.cu -- SURVEY §8(f) NEXT #3: GPU-side frontier sampling (Alg. 2, PAPER.md:366-385,
// reading R9) and induced-subgraph extraction (Alg. 2 line 9), `count` samplers at once (the
// paper's inter-sampler parallelism).
//
// Alg. 2 is inherently sequential inside one sampler (every pop changes the frontier
// distribution), so one warp runs one sampler: lane 0 owns the frontier in shared memory with
// a Fenwick tree over the frontier degrees (degree-proportional pop in O(log m), "dynamic
// probability distribution"), and the parent graph's CSR is read from L2/HBM. Independent
// samplers fill the GPU. Induction is data-parallel: V_s lives as a bitmap over the parent, its
// ascending local ids are prefix popcounts, and each (sample, node) warp compacts the parent
// neighbor list with ballots -- rows come out ascending because the parent rows are ascending
// and the rank map is monotone (the precondition of Alg. 4).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

struct gsg_parent {
  int device = 0;
  int64_t N = 0, nnz = 0;
  int64_t* indptr = nullptr;
  int32_t* indices = nullptr;
  int32_t* noniso = nullptr;  // ascending non-isolated node ids
  int64_t n_noniso = 0;
  int64_t max_deg = 0;
};

struct gsg_sample {
  int device = 0;
  gsg_ctx* owner = nullptr;    // context whose spare pool receives the arrays at gsg_sample_free
  size_t nodes_bytes = 0, indptr_bytes = 0, indices_bytes = 0;
  int count = 0, n_cap = 0;
  std::vector<int32_t> n_k;
  std::vector<int64_t> nnz_k, idx_off;
  int32_t* nodes = nullptr;    // [count][n_cap]
  int64_t* indptr = nullptr;   // [count][n_cap + 1]
  int32_t* indices = nullptr;  // concatenated
  int32_t* d_n = nullptr;      // [count] n_k on the device (gsg_sample_load)
  int64_t* d_idx_off = nullptr;  // [count] offset of sample k in indices
  int32_t* d_err = nullptr;    // gsg_sample_load: a sample did not fit the subgraph (checked by gsg_sample_check)
};

namespace gsg {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t rng(uint64_t seed, uint64_t i, uint32_t j) { return mix64(seed ^ mix64(4 * i + j)); }
__device__ __forceinline__ uint32_t below(uint64_t r, uint32_t N) { return (uint32_t)(((r >> 32) * (uint64_t)N) >> 32); }

__device__ __forceinline__ bool bit_get(const uint32_t* b, int64_t v) { return (b[v >> 5] >> (v & 31)) & 1u; }

// 32-bit shared-window accesses for the frontier state (the descent below is a chain of
// dependent shared loads: generic addressing re-derived the window every step).
template <typename T> __device__ __forceinline__ T lds(uint32_t a);
template <> __device__ __forceinline__ int32_t lds<int32_t>(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
template <> __device__ __forceinline__ int64_t lds<int64_t>(uint32_t a) {
  int64_t v;
  asm volatile("ld.shared.s64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, int32_t v) { asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
__device__ __forceinline__ void sts(uint32_t a, int64_t v) { asm volatile("st.shared.s64 [%0], %1;" ::"r"(a), "l"(v) : "memory"); }

// One warp per sampler; lane 0 runs Alg. 2. Shared memory holds the frontier's degrees, row
// starts and a Fenwick tree over the degrees (FenT / StartT: int32 whenever the frontier degree
// sum / the parent's entry count fit: 36 KB at m = 3000, so ~6 samplers share an SM instead of
// 2). The V_s membership test of iteration i's new node (a bitmap word in global memory) is
// issued at the end of iteration i and consumed only after iteration i+1's neighbor pick has
// been issued, so the two global accesses overlap; if consuming it completes V_s, iteration
// i+1 is abandoned before it changes any state -- the sampled set is exactly the serial Alg. 2's.
template <typename FenT, typename StartT>
__global__ void k_frontier(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                           const int32_t* __restrict__ noniso, int64_t n_noniso, int n, int m, int clip,
                           uint64_t seed, int64_t words, uint32_t* __restrict__ bitmaps, int32_t* __restrict__ vs_all,
                           int32_t* __restrict__ nv_out) {
  extern __shared__ int64_t sm64[];
  FenT* fen = reinterpret_cast<FenT*>(sm64);                                    // [m + 1]
  StartT* fstart = reinterpret_cast<StartT*>(fen + (m + 1 + 1) / 2 * 2);        // [m] (8-byte aligned)
  int32_t* fdeg = reinterpret_cast<int32_t*>(fstart + (m + 1) / 2 * 2);         // [m]
  const uint32_t fen_s = (uint32_t)__cvta_generic_to_shared(fen);
  const uint32_t fstart_s = (uint32_t)__cvta_generic_to_shared(fstart);
  const uint32_t fdeg_s = (uint32_t)__cvta_generic_to_shared(fdeg);
  const int s = blockIdx.x;
  const int lane = threadIdx.x;
  const uint64_t sd = mix64(mix64(seed) + (uint64_t)s);  // gsg.h: seed_k (decorrelated across calls)
  uint32_t* bits = bitmaps + (int64_t)s * words;
  int32_t* vs = vs_all + (int64_t)s * n;
  // FS_0: m distinct nodes, uniform over the non-isolated nodes (attempt counter t). The
  // candidates c_t do not depend on the state, so the warp draws 32 attempts at once; attempt t
  // is accepted iff c_t is not in V_s yet and no earlier attempt of the batch drew it, and only
  // the first m - cnt acceptances count -- exactly the serial rejection loop.
  int cnt = 0;
  for (uint64_t t0 = 0; cnt < m; t0 += 32) {
    const int32_t c = noniso[below(rng(sd, t0 + lane, 3), (uint32_t)n_noniso)];
    const unsigned same = __match_any_sync(0xffffffffu, c);
    const bool fresh = !bit_get(bits, c) && !(same & ((1u << lane) - 1u));
    const unsigned acc = __ballot_sync(0xffffffffu, fresh);
    const int rank = __popc(acc & ((1u << lane) - 1u));
    const int need = m - cnt;
    if (fresh && rank < need) {
      atomicOr(&bits[c >> 5], 1u << (c & 31));
      const int64_t b0 = indptr[c];
      fstart[cnt + rank] = (StartT)b0;
      fdeg[cnt + rank] = (int32_t)(indptr[c + 1] - b0);
      vs[cnt + rank] = c;
    }
    cnt += min(__popc(acc), need);
    __syncwarp();
  }
  __threadfence_block();
  if (lane != 0) return;
  // Fenwick tree over the frontier degrees (1-based)
  FenT total = 0;
  for (int i = 1; i <= m; i++) { fen[i] = fdeg[i - 1]; total += fdeg[i - 1]; }
  for (int i = 1; i <= m; i++) {
    const int j = i + (i & -i);
    if (j <= m) fen[j] += fen[i];
  }
  int top = 1;
  while (top * 2 <= m) top *= 2;
  int nv = m;
  const uint64_t max_it = 1000ull * n + 1000000ull;
  int32_t pend = -1;   // new frontier node of the previous iteration, membership not yet tested
  uint32_t pword = 0;  // its bitmap word (load in flight)
  for (uint64_t it = 0; nv < n; it++) {
    if (it == max_it) break;
    // Alg. 2 line 4: slot with probability deg(u) / sum_FS deg  (smallest slot with prefix > x)
    FenT x = (FenT)below(rng(sd, it, 0), (uint32_t)total);
    const uint64_t r1 = rng(sd, it, 1);
    int pos = 0;
#pragma unroll
    for (int lv = 13; lv >= 0; lv--) {  // m <= 16384: top <= 2^13
      const int step = 1 << lv;
      if (step <= top && pos + step <= m) {
        const FenT v = lds<FenT>(fen_s + (uint32_t)(pos + step) * sizeof(FenT));
        if (v <= x) { pos += step; x -= v; }
      }
    }
    const int slot = pos;
    const int32_t du = lds<int32_t>(fdeg_s + 4u * slot);
    // line 5: uniform neighbor u' of u
    const int32_t up = indices[(int64_t)lds<StartT>(fstart_s + (uint32_t)sizeof(StartT) * slot) + below(r1, (uint32_t)du)];
    const int64_t bu = indptr[up], eu = indptr[up + 1];
    // R9: the previous iteration's new frontier node joins V_s (tested while u' is in flight)
    if (pend >= 0) {
      if (!((pword >> (pend & 31)) & 1u)) {
        // pword is the word's current value (loaded after every earlier set; only this thread
        // writes this sampler's bitmap): a plain store, no dependent read-modify-write
        bits[pend >> 5] = pword | (1u << (pend & 31));
        vs[nv++] = pend;
      }
      pend = -1;
      if (nv >= n) break;  // V_s complete: this iteration never happened
    }
    // line 6: FS <- FS \ {u} U {u'}
    const int32_t dup = (int32_t)(eu - bu);
    sts(fstart_s + (uint32_t)sizeof(StartT) * slot, (StartT)bu);
    sts(fdeg_s + 4u * slot, dup);
    const FenT delta = (FenT)dup - (FenT)du;
    for (int i = slot + 1; i <= m; i += i & -i) {
      const uint32_t a = fen_s + (uint32_t)i * sizeof(FenT);
      sts(a, (FenT)(lds<FenT>(a) + delta));
    }
    total += delta;
    pend = up;
    pword = bits[up >> 5];
  }
  if (pend >= 0 && nv < n && !((pword >> (pend & 31)) & 1u)) {  // the last iteration's test (max_it)
    bits[pend >> 5] |= 1u << (pend & 31);
    vs[nv++] = pend;
  }
  // clipping to a multiple of `clip` by uniformly random removals
  const int keep = nv / clip * clip;
  for (uint64_t r = 0; nv > keep; r++) {
    const int j = (int)below(rng(sd, r, 2), (uint32_t)nv);
    const int32_t v = vs[j];
    bits[v >> 5] &= ~(1u << (v & 31));
    vs[j] = vs[nv - 1];
    nv--;
  }
  nv_out[s] = nv;
}

// Per sampler (one block): exclusive prefix of the bitmap's popcounts (the local id of the first
// node of each word) and the ascending node list.
__global__ void k_rank(const uint32_t* __restrict__ bitmaps, int64_t words, int n_cap, int32_t* __restrict__ wordpre,
                       int32_t* __restrict__ nodes_all) {
  __shared__ int32_t part[1024];
  const int s = blockIdx.x;
  const uint32_t* bits = bitmaps + (int64_t)s * words;
  int32_t* pre = wordpre + (int64_t)s * words;
  int32_t* nodes = nodes_all + (int64_t)s * n_cap;
  const int64_t per = (words + blockDim.x - 1) / blockDim.x;
  const int64_t w0 = threadIdx.x * per, w1 = min(words, w0 + per);
  int32_t sum = 0;
  for (int64_t w = w0; w < w1; w++) sum += __popc(bits[w]);
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {  // inclusive Hillis-Steele scan
    const int32_t v = threadIdx.x >= (unsigned)off ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int32_t run = part[threadIdx.x] - sum;
  for (int64_t w = w0; w < w1; w++) {
    pre[w] = run;
    uint32_t b = bits[w];
    while (b) {
      const int t = __ffs(b) - 1;
      if (run < n_cap) nodes[run] = (int32_t)(w * 32 + t);
      run++;
      b &= b - 1;
    }
  }
}

// Warp per (sample, local node): number of parent neighbors inside V_s.
__global__ void k_rowcount(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                           const uint32_t* __restrict__ bitmaps, int64_t words, const int32_t* __restrict__ nodes_all,
                           const int32_t* __restrict__ nv, int count, int n_cap, int32_t* __restrict__ rowcnt_all) {
  const int lane = threadIdx.x & 31;
  const int64_t total = (int64_t)count * n_cap;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < total;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int s = (int)(t / n_cap), i = (int)(t % n_cap);
    if (i >= nv[s]) continue;
    const uint32_t* bits = bitmaps + (int64_t)s * words;
    const int32_t v = nodes_all[(int64_t)s * n_cap + i];
    int c = 0;
    for (int64_t k0 = indptr[v]; k0 < indptr[v + 1]; k0 += 32) {
      const int64_t k = k0 + lane;
      const bool hit = k < indptr[v + 1] && bit_get(bits, indices[k]);
      c += __popc(__ballot_sync(0xffffffffu, hit));
    }
    if (lane == 0) rowcnt_all[(int64_t)s * n_cap + i] = c;
  }
}

// Per sampler (one block): indptr = exclusive scan of the row counts.
__global__ void k_rowscan(int n_cap, const int32_t* __restrict__ nv, const int32_t* __restrict__ rowcnt_all,
                          int64_t* __restrict__ indptr_all) {
  __shared__ int64_t part[1024];
  const int s = blockIdx.x;
  const int n = nv[s];
  int64_t* ip = indptr_all + (int64_t)s * (n_cap + 1);
  const int32_t* rc = rowcnt_all + (int64_t)s * n_cap;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int r0 = threadIdx.x * per, r1 = min(n, r0 + per);
  int64_t sum = 0;
  for (int r = r0; r < r1; r++) sum += rc[r];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {
    const int64_t v = threadIdx.x >= (unsigned)off ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t run = part[threadIdx.x] - sum;
  for (int r = r0; r < r1; r++) {
    ip[r] = run;
    run += rc[r];
  }
  __syncthreads();
  if (threadIdx.x == blockDim.x - 1 || (threadIdx.x == 0 && n == 0)) ip[n] = part[blockDim.x - 1];
}

// Warp per (sample, local node): write the local ids of the in-V_s neighbors, ascending.
__global__ void k_induce_fill(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                              const uint32_t* __restrict__ bitmaps, int64_t words, const int32_t* __restrict__ wordpre,
                              const int32_t* __restrict__ nodes_all, const int32_t* __restrict__ nv, int count,
                              int n_cap, const int64_t* __restrict__ sub_indptr_all, const int64_t* __restrict__ idx_off,
                              int32_t* __restrict__ sub_indices) {
  const int lane = threadIdx.x & 31;
  const int64_t total = (int64_t)count * n_cap;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < total;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int s = (int)(t / n_cap), i = (int)(t % n_cap);
    if (i >= nv[s]) continue;
    const uint32_t* bits = bitmaps + (int64_t)s * words;
    const int32_t* pre = wordpre + (int64_t)s * words;
    const int32_t v = nodes_all[(int64_t)s * n_cap + i];
    int32_t* out = sub_indices + idx_off[s] + sub_indptr_all[(int64_t)s * (n_cap + 1) + i];
    int o = 0;
    for (int64_t k0 = indptr[v]; k0 < indptr[v + 1]; k0 += 32) {
      const int64_t k = k0 + lane;
      const int32_t w = k < indptr[v + 1] ? indices[k] : 0;
      const bool hit = k < indptr[v + 1] && bit_get(bits, w);
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const uint32_t word = bits[w >> 5];
        out[o + __popc(m & ((1u << lane) - 1))] = pre[w >> 5] + __popc(word & ((1u << (w & 31)) - 1));
      }
      o += __popc(m);
    }
  }
}

// Induction with the sampler's V_s bitmap in SHARED memory (one 1024-thread block per sample):
// the global-bitmap kernels above test every parent neighbor of every sampled node against a
// 200 KB-per-sample bitmap that, for hundreds of samples, no longer fits the L2 (2/3 of a
// sampling call went there). Count pass: per-row hit counts, then the exclusive scan into the
// sample's indptr. Fill pass: the same scan writing local ids, ranked through a uint16 prefix per
// 4-word group (local ids < 65536) plus at most 3 word popcounts. Used when the bitmap and the
// group prefixes fit in shared memory (parents up to ~1.6M nodes) and n < 65536.
constexpr int kInduceThreads = 1024;

__device__ __forceinline__ void load_bitmap_smem(const uint32_t* __restrict__ bits, int64_t words, uint32_t* sb) {
  for (int64_t w = threadIdx.x; w < words; w += blockDim.x) sb[w] = bits[w];
}

__device__ __forceinline__ bool sbit(const uint32_t* sb, int32_t v) { return (sb[v >> 5] >> (v & 31)) & 1u; }

// The count pass's adjacency scan: lane l reads parent-neighbor entries [k0 + 4 l, k0 + 4 l + 4)
// with one 16-byte load (k0 a multiple of 4: the parent's index array is padded by 4 entries),
// kIU such loads in flight per lane, and the next node's row range is fetched while the current
// row is scanned (888 config-5 samples: 26.3 -> 21.5 ms). The same scheme in the fill pass (int4
// loads with a warp scan of the hit counts, or 8 four-byte loads per lane in flight) was slower
// there (94 / 66 vs 60 ms; with four ballots per 16-byte group instead of the scan 56 vs 52 ms):
// its cost is the ranking of the hits in shared memory and their stores, not the loads.
constexpr int kIU = 4;

__device__ __forceinline__ unsigned hit_bits(const uint32_t* sb, int4 w, int64_t k, int64_t b, int64_t e) {
  unsigned h = 0;
  h |= (k + 0 >= b && k + 0 < e && sbit(sb, w.x)) ? 1u : 0u;
  h |= (k + 1 >= b && k + 1 < e && sbit(sb, w.y)) ? 2u : 0u;
  h |= (k + 2 >= b && k + 2 < e && sbit(sb, w.z)) ? 4u : 0u;
  h |= (k + 3 >= b && k + 3 < e && sbit(sb, w.w)) ? 8u : 0u;
  return h;
}

// Visits the sample's nodes i = warp, warp + 32, ... with their parent row [b, e); body(i, b, e).
template <typename Body>
__device__ __forceinline__ void for_each_row(const int64_t* __restrict__ indptr, const int32_t* __restrict__ nodes,
                                             int n, int warp, Body body) {
  constexpr int NW = kInduceThreads / 32;
  if (warp >= n) return;
  int32_t v = nodes[warp];
  int64_t b = indptr[v], e = indptr[v + 1];
  int32_t v1 = warp + NW < n ? nodes[warp + NW] : 0;
  for (int i = warp; i < n; i += NW) {
    int64_t b1 = 0, e1 = 0;
    int32_t v2 = 0;
    if (i + NW < n) {  // next row's range and the row after it: in flight during this row's scan
      b1 = indptr[v1];
      e1 = indptr[v1 + 1];
      if (i + 2 * NW < n) v2 = nodes[i + 2 * NW];
    }
    body(i, b, e);
    b = b1;
    e = e1;
    v1 = v2;
  }
}

__global__ void __launch_bounds__(kInduceThreads) k_induce_count_smem(const int64_t* __restrict__ indptr,
                                                                      const int32_t* __restrict__ indices,
                                                                      const uint32_t* __restrict__ bitmaps, int64_t words,
                                                                      const int32_t* __restrict__ nodes_all,
                                                                      const int32_t* __restrict__ nv, int n_cap,
                                                                      int32_t* __restrict__ rowcnt_all,
                                                                      int64_t* __restrict__ indptr_all) {
  extern __shared__ uint32_t sb[];
  __shared__ int64_t part[32];
  const int s = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  load_bitmap_smem(bitmaps + (int64_t)s * words, words, sb);
  __syncthreads();
  const int n = nv[s];
  const int32_t* nodes = nodes_all + (int64_t)s * n_cap;
  int32_t* rc = rowcnt_all + (int64_t)s * n_cap;
  for_each_row(indptr, nodes, n, warp, [&](int i, int64_t b, int64_t e) {
    int c = 0;
    for (int64_t k0 = b & ~3LL; k0 < e; k0 += 128 * kIU) {
      int4 w[kIU];
#pragma unroll
      for (int q = 0; q < kIU; q++) {
        const int64_t k = k0 + 128 * q + 4 * lane;
        w[q] = k < e ? __ldg(reinterpret_cast<const int4*>(indices + k)) : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int q = 0; q < kIU; q++) c += __popc(hit_bits(sb, w[q], k0 + 128 * q + 4 * lane, b, e));
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) rc[i] = c;
  });
  __syncthreads();
  // indptr = exclusive scan of the row counts (rows split into equal runs per thread)
  int64_t* ip = indptr_all + (int64_t)s * (n_cap + 1);
  const int per = (n + kInduceThreads - 1) / kInduceThreads;
  const int r0 = threadIdx.x * per, r1 = min(n, r0 + per);
  int64_t sum = 0;
  for (int r = r0; r < r1; r++) sum += rc[r];
  int64_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) part[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t t = part[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += u;
    }
    part[lane] = t;
  }
  __syncthreads();
  int64_t run = (warp > 0 ? part[warp - 1] : 0) + incl - sum;
  for (int r = r0; r < r1; r++) {
    ip[r] = run;
    run += rc[r];
  }
  if (threadIdx.x == 0) ip[n] = part[31];
}

__global__ void __launch_bounds__(kInduceThreads) k_induce_fill_smem(const int64_t* __restrict__ indptr,
                                                                     const int32_t* __restrict__ indices,
                                                                     const uint32_t* __restrict__ bitmaps, int64_t words,
                                                                     const int32_t* __restrict__ nodes_all,
                                                                     const int32_t* __restrict__ nv, int n_cap,
                                                                     const int64_t* __restrict__ sub_indptr_all,
                                                                     const int64_t* __restrict__ idx_off,
                                                                     int32_t* __restrict__ sub_indices) {
  extern __shared__ uint32_t sb[];
  __shared__ int32_t part[32];
  const int s = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  load_bitmap_smem(bitmaps + (int64_t)s * words, words, sb);
  uint16_t* gp = reinterpret_cast<uint16_t*>(sb + words);  // [ceil(words / 4)] rank before each 4-word group
  const int64_t groups = (words + 3) / 4;
  __syncthreads();
  {  // group prefixes: each thread a contiguous run of groups, block scan of the run sums
    const int64_t per = (groups + kInduceThreads - 1) / kInduceThreads;
    const int64_t g0 = threadIdx.x * per, g1 = min(groups, g0 + per);
    int32_t sum = 0;
    for (int64_t g = g0; g < g1; g++)
      for (int64_t w = 4 * g; w < min(words, 4 * g + 4); w++) sum += __popc(sb[w]);
    int32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) part[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int32_t t = part[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t u = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += u;
      }
      part[lane] = t;
    }
    __syncthreads();
    int32_t run = (warp > 0 ? part[warp - 1] : 0) + incl - sum;
    for (int64_t g = g0; g < g1; g++) {
      gp[g] = (uint16_t)run;
      for (int64_t w = 4 * g; w < min(words, 4 * g + 4); w++) run += __popc(sb[w]);
    }
  }
  __syncthreads();
  const int n = nv[s];
  const int32_t* nodes = nodes_all + (int64_t)s * n_cap;
  const int64_t* sip = sub_indptr_all + (int64_t)s * (n_cap + 1);
  int32_t* outb = sub_indices + idx_off[s];
  for (int i = warp; i < n; i += kInduceThreads / 32) {
    const int32_t v = nodes[i];
    const int64_t b = indptr[v], e = indptr[v + 1];
    int32_t* out = outb + sip[i];
    int o = 0;
    for (int64_t k0 = b; k0 < e; k0 += 128) {
      int32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; q++) w[q] = k0 + 32 * q + lane < e ? indices[k0 + 32 * q + lane] : -1;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const bool hit = w[q] >= 0 && sbit(sb, w[q]);
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          // rank = the group's prefix + the bits below v in its 4-word group, read as ONE 16-byte
          // load (the words past the bitmap's end that a last group may cover lie above v)
          const int32_t wd = w[q] >> 5, j = wd & 3;
          const uint4 g4 = reinterpret_cast<const uint4*>(sb)[wd >> 2];
          const uint32_t below = (1u << (w[q] & 31)) - 1;
          int32_t r = gp[wd >> 2];
          r += j > 0 ? __popc(g4.x) : __popc(g4.x & below);
          if (j >= 1) r += j > 1 ? __popc(g4.y) : __popc(g4.y & below);
          if (j >= 2) r += j > 2 ? __popc(g4.z) : __popc(g4.z & below);
          if (j >= 3) r += __popc(g4.w & below);
          out[o + __popc(m & ((1u << lane) - 1))] = r;
        }
        o += __popc(m);
      }
    }
  }
}

// nnz_k = indptr_k[n_k] of every sample, gathered for ONE device -> host copy
__global__ void k_sample_nnz(int count, int n_cap, const int64_t* __restrict__ indptr_all,
                             const int32_t* __restrict__ nv, int64_t* __restrict__ nnz) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < count; k += gridDim.x * blockDim.x)
    nnz[k] = indptr_all[(int64_t)k * (n_cap + 1) + nv[k]];
}

// gsg_sample_load: sample *d_k into a device-sized subgraph of n_pad nodes. Nodes n_k .. n_pad-1
// are isolated padding (empty rows; normalization gives them a self loop, their feature rows are
// gathered as zeros and their loss weight is 0), so one CUDA graph of the step serves every
// sample: every size the kernels need is read from device memory.
__global__ void k_sample_load(const int32_t* __restrict__ d_k, int n_cap, const int32_t* __restrict__ s_n,
                              const int64_t* __restrict__ s_indptr, const int64_t* __restrict__ s_off,
                              const int32_t* __restrict__ s_indices, const int32_t* __restrict__ s_nodes, int n_pad,
                              int64_t nnz_cap, int64_t* __restrict__ indptr, int32_t* __restrict__ indices,
                              int32_t* __restrict__ nodes_out, float* __restrict__ node_w, int32_t* __restrict__ err) {
  const int k = *d_k;
  const int nk = s_n[k];
  const int64_t* ip = s_indptr + (int64_t)k * (n_cap + 1);
  const int64_t nnz = ip[nk];
  if (nk > n_pad || nnz > nnz_cap) {  // does not fit: leave the subgraph empty and flag it
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(err, 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n_pad; i += (int64_t)gridDim.x * blockDim.x)
      indptr[i] = 0;
    return;
  }
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const float w = nk > 0 ? 1.0f / (float)nk : 0.f;
  for (int64_t i = t0; i <= n_pad; i += T) {
    indptr[i] = i <= nk ? ip[i] : nnz;
    if (i < n_pad) {
      const bool real = i < nk;
      if (nodes_out) nodes_out[i] = real ? s_nodes[(int64_t)k * n_cap + i] : -1;
      if (node_w) node_w[i] = real ? w : 0.f;
    }
  }
  const int32_t* src = s_indices + s_off[k];
  for (int64_t e0 = t0; e0 < nnz; e0 += 4 * T) {  // 4 loads in flight per thread
    int32_t v[4];
#pragma unroll
    for (int u = 0; u < 4; u++) v[u] = e0 + u * T < nnz ? __ldg(src + e0 + u * T) : 0;
#pragma unroll
    for (int u = 0; u < 4; u++)
      if (e0 + u * T < nnz) indices[e0 + u * T] = v[u];
  }
}

__global__ void k_advance(int32_t* d_k, int count) { *d_k = (*d_k + 1) % count; }

}  // namespace
}  // namespace gsg

using namespace gsg;

namespace gsg {
// A device buffer of at least `bytes` for a sample array: the smallest spare of the context that
// fits and is not more than twice as large, else a fresh allocation.
static cudaError_t pool_take(gsg_ctx* c, size_t bytes, void** out, size_t* got) {
  int best = -1;
  for (int i = 0; i < (int)c->spare.size(); i++) {
    const size_t b = c->spare[i].second;
    if (b >= bytes && b <= 2 * bytes + (1u << 20) && (best < 0 || b < c->spare[best].second)) best = i;
  }
  if (best >= 0) {
    *out = c->spare[best].first;
    *got = c->spare[best].second;
    c->spare.erase(c->spare.begin() + best);
    return cudaSuccess;
  }
  *got = bytes;
  return cudaMalloc(out, bytes);
}

// Back to the context's spare list (at most kSpare buffers are kept: the smallest goes).
static void pool_give(gsg_ctx* c, void* p, size_t bytes) {
  constexpr size_t kSpare = 8;
  if (!p) return;
  if (!c) { cudaFree(p); return; }
  c->spare.emplace_back(p, bytes);
  if (c->spare.size() > kSpare) {
    size_t m = 0;
    for (size_t i = 1; i < c->spare.size(); i++)
      if (c->spare[i].second < c->spare[m].second) m = i;
    cudaFree(c->spare[m].first);
    c->spare.erase(c->spare.begin() + m);
  }
}

void sampler_detach(gsg_ctx* c) {
  for (gsg_sample* s : c->live_samples) s->owner = nullptr;
  c->live_samples.clear();
}
}  // namespace gsg

extern "C" {

GSG_API int gsg_parent_upload(gsg_ctx_t c, int64_t N, int64_t nnz, const int64_t* h_indptr, const int32_t* h_indices,
                              gsg_parent_t* out) {
  GSG_CHECK(c && out && h_indptr && (nnz == 0 || h_indices), GSG_EINVAL, "NULL argument");
  GSG_CHECK(N >= 1 && N < INT32_MAX && nnz >= 0, GSG_EINVAL, "bad parent sizes N=%lld nnz=%lld", (long long)N,
            (long long)nnz);
  GSG_CHECK(h_indptr[N] == nnz, GSG_EGRAPH, "indptr[N] != nnz");
  DeviceGuard dg(c->device);
  std::vector<int32_t> non;
  non.reserve(N);
  for (int64_t i = 0; i < N; i++)
    if (h_indptr[i + 1] > h_indptr[i]) non.push_back((int32_t)i);
  auto* p = new gsg_parent;
  p->device = c->device;
  p->N = N;
  p->nnz = nnz;
  p->n_noniso = (int64_t)non.size();
  for (int64_t i = 0; i < N; i++) p->max_deg = std::max<int64_t>(p->max_deg, h_indptr[i + 1] - h_indptr[i]);
  cudaError_t e = cudaMalloc(&p->indptr, sizeof(int64_t) * (N + 1));
  // 4 entries of padding: the induction scans read whole 16-byte groups (their tails masked)
  if (e == cudaSuccess) e = cudaMalloc(&p->indices, sizeof(int32_t) * (nnz + 4));
  if (e == cudaSuccess) e = cudaMalloc(&p->noniso, sizeof(int32_t) * (non.size() > 0 ? non.size() : 1));
  if (e == cudaSuccess) e = cudaMemcpy(p->indptr, h_indptr, sizeof(int64_t) * (N + 1), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && nnz) e = cudaMemcpy(p->indices, h_indices, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !non.empty())
    e = cudaMemcpy(p->noniso, non.data(), sizeof(int32_t) * non.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    gsg_parent_free(p);
    return cuda_fail(e, "gsg_parent_upload");
  }
  *out = p;
  return GSG_OK;
}

GSG_API int gsg_parent_free(gsg_parent_t p) {
  if (!p) return GSG_OK;
  DeviceGuard dg(p->device);
  cudaFree(p->indptr);
  cudaFree(p->indices);
  cudaFree(p->noniso);
  delete p;
  return GSG_OK;
}

GSG_API int gsg_frontier_sample(gsg_ctx_t c, gsg_parent_t p, int32_t n, int32_t m, int32_t clip, uint64_t seed,
                                int32_t count, gsg_sample_t* out) {
  NvtxRange nvtx("gsg sampler frontier_sample");
  GSG_CHECK(c && p && out, GSG_EINVAL, "NULL argument");
  GSG_CHECK(count >= 1 && m >= 1 && m <= n && m <= 16384 && clip >= 1, GSG_EINVAL,
            "bad sampler sizes n=%d m=%d clip=%d count=%d", n, m, clip, count);
  GSG_CHECK((int64_t)n <= p->n_noniso && (int64_t)m <= p->n_noniso, GSG_EINVAL,
            "n=%d / m=%d exceed the parent's %lld non-isolated nodes", n, m, (long long)p->n_noniso);
  DeviceGuard dg(c->device);
  cudaStream_t st = c->stream;
  const int64_t words = (p->N + 31) / 32;
  // scratch of this call: context workspaces, grown on demand and kept
  DevBuf &bitmaps = c->ws_sbits, &vs = c->ws_svs, &nv = c->ws_snv, &wordpre = c->ws_swordpre, &nnzb = c->ws_snnz;
  int rc;
  if ((rc = bitmaps.reserve(sizeof(uint32_t) * words * count))) return rc;
  if ((rc = vs.reserve(sizeof(int32_t) * (int64_t)n * count))) return rc;
  if ((rc = nv.reserve(sizeof(int32_t) * count))) return rc;
  if ((rc = wordpre.reserve(sizeof(int32_t) * words * count))) return rc;
  if ((rc = nnzb.reserve(sizeof(int64_t) * count))) return rc;
  auto* S = new gsg_sample;
  S->device = c->device;
  S->owner = c;
  c->live_samples.push_back(S);
  S->count = count;
  S->n_cap = n;
  auto cleanup = [&](int code) {
    gsg_sample_free(S);
    return code;
  };
  cudaError_t e = pool_take(c, sizeof(int32_t) * (int64_t)n * count, (void**)&S->nodes, &S->nodes_bytes);
  if (e == cudaSuccess)
    e = pool_take(c, sizeof(int64_t) * (int64_t)(n + 1) * count, (void**)&S->indptr, &S->indptr_bytes);
  if (e != cudaSuccess) return cleanup(cuda_fail(e, "cudaMalloc(sample)"));
  e = cudaMemsetAsync(bitmaps.ptr, 0, sizeof(uint32_t) * words * count, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(S->indptr, 0, sizeof(int64_t) * (int64_t)(n + 1) * count, st);
  if (e != cudaSuccess) return cleanup(cuda_fail(e, "cudaMemsetAsync(sample)"));
  // frontier state: 4-byte Fenwick sums / row starts whenever they fit (36 KB for m = 3000:
  // ~6 samplers per SM), else 8-byte ones
  const bool fen32 = (int64_t)m * p->max_deg < (int64_t)INT32_MAX, start32 = p->nnz < (int64_t)INT32_MAX;
  const size_t mm = (size_t)(m + 1) / 2 * 2 + 2;
  const size_t smem = mm * (fen32 ? 4 : 8) + mm * (start32 ? 4 : 8) + 4 * (size_t)m + 16;
  auto launch = [&](auto kern) {
    cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (r != cudaSuccess) return r;
    kern<<<count, 32, smem, st>>>(p->indptr, p->indices, p->noniso, p->n_noniso, n, m, clip,
                                  seed, words, (uint32_t*)bitmaps.ptr, (int32_t*)vs.ptr, (int32_t*)nv.ptr);
    return cudaGetLastError();
  };
  if (fen32 && start32) e = launch(k_frontier<int32_t, int32_t>);
  else if (start32) e = launch(k_frontier<int64_t, int32_t>);
  else if (fen32) e = launch(k_frontier<int32_t, int64_t>);
  else e = launch(k_frontier<int64_t, int64_t>);
  if (e != cudaSuccess) return cleanup(cuda_fail(e, "k_frontier"));
  k_rank<<<count, 1024, 0, st>>>((const uint32_t*)bitmaps.ptr, words, n, (int32_t*)wordpre.ptr, S->nodes);
  const int64_t warps = (int64_t)count * n;
  int grid = (int)std::min<int64_t>((warps * 32 + 255) / 256, (int64_t)c->num_sms * 16);
  // row counts reuse the V_s insertion-order buffer (no longer needed after k_rank)
  // shared-memory induction when the V_s bitmap (+ uint16 group prefixes) fits one block
  const size_t ind_smem = sizeof(uint32_t) * (size_t)words + sizeof(uint16_t) * (size_t)((words + 3) / 4) + 16;
  static const int ind_env = getenv("GSG_SAMPLER_SMEM_INDUCE") ? atoi(getenv("GSG_SAMPLER_SMEM_INDUCE")) : 1;
  const bool smem_ind = ind_env && n < 65536 && ind_smem <= 225u * 1024u;
  if (smem_ind) {
    e = cudaFuncSetAttribute(k_induce_count_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ind_smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_induce_fill_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ind_smem);
    if (e != cudaSuccess) return cleanup(cuda_fail(e, "cudaFuncSetAttribute(induce)"));
    k_induce_count_smem<<<count, kInduceThreads, ind_smem, st>>>(p->indptr, p->indices, (const uint32_t*)bitmaps.ptr,
                                                                  words, S->nodes, (const int32_t*)nv.ptr, n,
                                                                  (int32_t*)vs.ptr, S->indptr);
    count_launch(c, 3);
  } else {
    k_rowcount<<<grid, 256, 0, st>>>(p->indptr, p->indices, (const uint32_t*)bitmaps.ptr, words, S->nodes,
                                     (const int32_t*)nv.ptr, count, n, (int32_t*)vs.ptr);
    k_rowscan<<<count, 1024, 0, st>>>(n, (const int32_t*)nv.ptr, (const int32_t*)vs.ptr, S->indptr);
    count_launch(c, 4);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return cleanup(cuda_fail(e, "sampler kernels"));
  // size the induced CSR arrays (the one host synchronization)
  S->n_k.resize(count);
  S->nnz_k.resize(count);
  S->idx_off.resize(count);
  k_sample_nnz<<<(count + 255) / 256, 256, 0, st>>>(count, n, S->indptr, (const int32_t*)nv.ptr,
                                                    (int64_t*)nnzb.ptr);
  count_launch(c);
  e = cudaMemcpyAsync(S->n_k.data(), nv.ptr, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(S->nnz_k.data(), nnzb.ptr, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cleanup(cuda_fail(e, "sampler sizes"));
  int64_t tot = 0;
  for (int k = 0; k < count; k++) {
    S->idx_off[k] = tot;
    tot += S->nnz_k[k];
  }
  e = pool_take(c, sizeof(int32_t) * (tot > 0 ? tot : 1), (void**)&S->indices, &S->indices_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&S->d_idx_off, sizeof(int64_t) * count);
  if (e == cudaSuccess) e = cudaMalloc(&S->d_n, sizeof(int32_t) * count);
  if (e == cudaSuccess) e = cudaMalloc(&S->d_err, sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMemsetAsync(S->d_err, 0, sizeof(int32_t), st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(S->d_idx_off, S->idx_off.data(), sizeof(int64_t) * count, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(S->d_n, nv.ptr, sizeof(int32_t) * count, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return cleanup(cuda_fail(e, "cudaMalloc(sample indices)"));
  if (smem_ind)
    k_induce_fill_smem<<<count, kInduceThreads, ind_smem, st>>>(p->indptr, p->indices, (const uint32_t*)bitmaps.ptr,
                                                                 words, S->nodes, (const int32_t*)nv.ptr, n, S->indptr,
                                                                 S->d_idx_off, S->indices);
  else
    k_induce_fill<<<grid, 256, 0, st>>>(p->indptr, p->indices, (const uint32_t*)bitmaps.ptr, words,
                                        (const int32_t*)wordpre.ptr, S->nodes, (const int32_t*)nv.ptr, count, n,
                                        S->indptr, S->d_idx_off, S->indices);
  count_launch(c);
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) {
    gsg_sample_free(S);
    return cuda_fail(e, "k_induce_fill");
  }
  *out = S;
  return GSG_OK;
}

GSG_API int gsg_sample_get(gsg_sample_t s, int32_t k, int32_t* n_k, int64_t* nnz_k, const int64_t** d_indptr,
                           const int32_t** d_indices, const int32_t** d_nodes) {
  GSG_CHECK(s && k >= 0 && k < s->count, GSG_EINVAL, "bad sample index %d", k);
  if (n_k) *n_k = s->n_k[k];
  if (nnz_k) *nnz_k = s->nnz_k[k];
  if (d_indptr) *d_indptr = s->indptr + (int64_t)k * (s->n_cap + 1);
  if (d_indices) *d_indices = s->indices + s->idx_off[k];
  if (d_nodes) *d_nodes = s->nodes + (int64_t)k * s->n_cap;
  return GSG_OK;
}

GSG_API int gsg_sample_load(gsg_ctx_t c, gsg_sample_t s, int32_t* d_k, gsg_subgraph_t sg, int32_t* d_nodes_out,
                            float* d_node_w) {
  NvtxRange nvtx("gsg sampler sample_load");
  GSG_CHECK(c && s && d_k && sg, GSG_EINVAL, "NULL argument");
  GSG_CHECK(sg->dev_sized, GSG_EINVAL, "gsg_sample_load needs a subgraph from gsg_subgraph_create_device");
  DeviceGuard dg(c->device);
  const int64_t work = std::max<int64_t>((int64_t)sg->n + 1, sg->cap_nnz);
  const int grid = (int)std::min<int64_t>((work + 255) / 256, (int64_t)c->num_sms * 8);
  k_sample_load<<<grid, 256, 0, c->stream>>>(d_k, s->n_cap, s->d_n, s->indptr, s->d_idx_off, s->indices, s->nodes,
                                             sg->n, sg->cap_nnz, sg->indptr, sg->indices, d_nodes_out, d_node_w,
                                             s->d_err);
  k_advance<<<1, 1, 0, c->stream>>>(d_k, s->count);
  count_launch(c, 2);
  sg->norm_mode = -1;
  GSG_CUDA(cudaGetLastError());
  return GSG_OK;
}

GSG_API int gsg_sample_check(gsg_sample_t s) {
  GSG_CHECK(s, GSG_EINVAL, "NULL sample");
  DeviceGuard dg(s->device);
  int32_t e = 0;
  GSG_CUDA(cudaMemcpy(&e, s->d_err, sizeof(int32_t), cudaMemcpyDeviceToHost));
  GSG_CHECK(e == 0, GSG_EINVAL, "gsg_sample_load: a sample exceeded the subgraph's node or entry capacity "
                                "(the subgraph was left empty for that step)");
  return GSG_OK;
}

GSG_API int gsg_sample_free(gsg_sample_t s) {
  if (!s) return GSG_OK;
  DeviceGuard dg(s->device);
  gsg_ctx* c = s->owner;
  if (c) {  // the big arrays go back to the context's spare list (reused by the next call)
    auto& L = c->live_samples;
    for (size_t i = 0; i < L.size(); i++)
      if (L[i] == s) { L.erase(L.begin() + i); break; }
    cudaDeviceSynchronize();  // as cudaFree would: no kernel may still read them when they are reused
  }
  pool_give(c, s->nodes, s->nodes_bytes);
  pool_give(c, s->indptr, s->indptr_bytes);
  pool_give(c, s->indices, s->indices_bytes);
  cudaFree(s->d_n);
  cudaFree(s->d_idx_off);
  cudaFree(s->d_err);
  delete s;
  return GSG_OK;
}

}  // extern "C"
