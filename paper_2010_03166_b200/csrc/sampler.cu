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
};

struct gsg_sample {
  int device = 0;
  int count = 0, n_cap = 0;
  std::vector<int32_t> n_k;
  std::vector<int64_t> nnz_k, idx_off;
  int32_t* nodes = nullptr;    // [count][n_cap]
  int64_t* indptr = nullptr;   // [count][n_cap + 1]
  int32_t* indices = nullptr;  // concatenated
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

// One warp per sampler; lane 0 runs Alg. 2. Shared: FS node ids, degrees, row starts, Fenwick.
__global__ void k_frontier(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                           const int32_t* __restrict__ noniso, int64_t n_noniso, int n, int m, int clip,
                           uint64_t seed, int64_t words, uint32_t* __restrict__ bitmaps, int32_t* __restrict__ vs_all,
                           int32_t* __restrict__ nv_out) {
  extern __shared__ int64_t sm64[];
  int64_t* fen = sm64;                                             // [m + 1]
  int64_t* fstart = fen + (m + 1);                                 // [m]
  int32_t* fnode = reinterpret_cast<int32_t*>(fstart + m);         // [m]
  int32_t* fdeg = fnode + m;                                       // [m]
  const int s = blockIdx.x;
  if (threadIdx.x != 0) return;
  const uint64_t sd = mix64(mix64(seed) + (uint64_t)s);  // gsg.h: seed_k (decorrelated across calls)
  uint32_t* bits = bitmaps + (int64_t)s * words;
  int32_t* vs = vs_all + (int64_t)s * n;
  // FS_0: m distinct nodes, uniform over the non-isolated nodes (attempt counter t)
  int cnt = 0;
  for (uint64_t t = 0; cnt < m; t++) {
    const int32_t c = noniso[below(rng(sd, t, 3), (uint32_t)n_noniso)];
    if (bit_get(bits, c)) continue;
    bits[c >> 5] |= 1u << (c & 31);
    const int64_t b0 = indptr[c];
    fnode[cnt] = c;
    fstart[cnt] = b0;
    fdeg[cnt] = (int32_t)(indptr[c + 1] - b0);
    vs[cnt] = c;
    cnt++;
  }
  // Fenwick tree over the frontier degrees (1-based)
  int64_t total = 0;
  for (int i = 1; i <= m; i++) { fen[i] = fdeg[i - 1]; total += fdeg[i - 1]; }
  for (int i = 1; i <= m; i++) {
    const int j = i + (i & -i);
    if (j <= m) fen[j] += fen[i];
  }
  int top = 1;
  while (top * 2 <= m) top *= 2;
  int nv = m;
  const uint64_t max_it = 1000ull * n + 1000000ull;
  for (uint64_t it = 0; nv < n && it < max_it; it++) {
    // Alg. 2 line 4: slot with probability deg(u) / sum_FS deg  (smallest slot with prefix > x)
    int64_t x = below(rng(sd, it, 0), (uint32_t)total);
    int pos = 0;
    for (int step = top; step > 0; step >>= 1) {
      if (pos + step <= m && fen[pos + step] <= x) { pos += step; x -= fen[pos]; }
    }
    const int slot = pos;
    const int32_t du = fdeg[slot];
    // line 5: uniform neighbor u' of u
    const int32_t up = indices[fstart[slot] + below(rng(sd, it, 1), (uint32_t)du)];
    const int64_t bu = indptr[up];
    const int32_t dup = (int32_t)(indptr[up + 1] - bu);
    // line 6: FS <- FS \ {u} U {u'}
    fnode[slot] = up;
    fstart[slot] = bu;
    fdeg[slot] = dup;
    const int64_t delta = (int64_t)dup - du;
    for (int i = slot + 1; i <= m; i += i & -i) fen[i] += delta;
    total += delta;
    // R9: the new frontier node joins V_s
    if (!bit_get(bits, up)) {
      bits[up >> 5] |= 1u << (up & 31);
      vs[nv++] = up;
    }
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

}  // namespace
}  // namespace gsg

using namespace gsg;

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
  cudaError_t e = cudaMalloc(&p->indptr, sizeof(int64_t) * (N + 1));
  if (e == cudaSuccess) e = cudaMalloc(&p->indices, sizeof(int32_t) * (nnz > 0 ? nnz : 1));
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
  GSG_CHECK(c && p && out, GSG_EINVAL, "NULL argument");
  GSG_CHECK(count >= 1 && m >= 1 && m <= n && m <= 16384 && clip >= 1, GSG_EINVAL,
            "bad sampler sizes n=%d m=%d clip=%d count=%d", n, m, clip, count);
  GSG_CHECK((int64_t)n <= p->n_noniso && (int64_t)m <= p->n_noniso, GSG_EINVAL,
            "n=%d / m=%d exceed the parent's %lld non-isolated nodes", n, m, (long long)p->n_noniso);
  DeviceGuard dg(c->device);
  cudaStream_t st = c->stream;
  const int64_t words = (p->N + 31) / 32;
  DevBuf bitmaps, vs, nv, wordpre;
  int rc;
  if ((rc = bitmaps.reserve(sizeof(uint32_t) * words * count))) return rc;
  if ((rc = vs.reserve(sizeof(int32_t) * (int64_t)n * count))) return rc;
  if ((rc = nv.reserve(sizeof(int32_t) * count))) return rc;
  if ((rc = wordpre.reserve(sizeof(int32_t) * words * count))) return rc;
  auto* S = new gsg_sample;
  S->device = c->device;
  S->count = count;
  S->n_cap = n;
  auto cleanup = [&](int code) {
    bitmaps.release(); vs.release(); nv.release(); wordpre.release();
    gsg_sample_free(S);
    return code;
  };
  cudaError_t e = cudaMalloc(&S->nodes, sizeof(int32_t) * (int64_t)n * count);
  if (e == cudaSuccess) e = cudaMalloc(&S->indptr, sizeof(int64_t) * (int64_t)(n + 1) * count);
  if (e != cudaSuccess) return cleanup(cuda_fail(e, "cudaMalloc(sample)"));
  e = cudaMemsetAsync(bitmaps.ptr, 0, sizeof(uint32_t) * words * count, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(S->indptr, 0, sizeof(int64_t) * (int64_t)(n + 1) * count, st);
  if (e != cudaSuccess) return cleanup(cuda_fail(e, "cudaMemsetAsync(sample)"));
  const size_t smem = sizeof(int64_t) * (2 * (size_t)m + 1) + sizeof(int32_t) * 2 * (size_t)m;
  e = cudaFuncSetAttribute(k_frontier, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cleanup(cuda_fail(e, "cudaFuncSetAttribute(k_frontier)"));
  k_frontier<<<count, 32, smem, st>>>(p->indptr, p->indices, p->noniso, p->n_noniso, n, m, clip, seed, words,
                                      (uint32_t*)bitmaps.ptr, (int32_t*)vs.ptr, (int32_t*)nv.ptr);
  k_rank<<<count, 1024, 0, st>>>((const uint32_t*)bitmaps.ptr, words, n, (int32_t*)wordpre.ptr, S->nodes);
  const int64_t warps = (int64_t)count * n;
  int grid = (int)std::min<int64_t>((warps * 32 + 255) / 256, (int64_t)c->num_sms * 16);
  // row counts reuse the V_s insertion-order buffer (no longer needed after k_rank)
  k_rowcount<<<grid, 256, 0, st>>>(p->indptr, p->indices, (const uint32_t*)bitmaps.ptr, words, S->nodes,
                                   (const int32_t*)nv.ptr, count, n, (int32_t*)vs.ptr);
  k_rowscan<<<count, 1024, 0, st>>>(n, (const int32_t*)nv.ptr, (const int32_t*)vs.ptr, S->indptr);
  count_launch(c, 4);
  if ((e = cudaGetLastError()) != cudaSuccess) return cleanup(cuda_fail(e, "sampler kernels"));
  // size the induced CSR arrays (the one host synchronization)
  S->n_k.resize(count);
  S->nnz_k.resize(count);
  S->idx_off.resize(count);
  e = cudaMemcpyAsync(S->n_k.data(), nv.ptr, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cleanup(cuda_fail(e, "sampler sizes"));
  int64_t tot = 0;
  for (int k = 0; k < count; k++) {
    int64_t v = 0;
    e = cudaMemcpy(&v, S->indptr + (int64_t)k * (n + 1) + S->n_k[k], sizeof(int64_t), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cleanup(cuda_fail(e, "sampler nnz"));
    S->nnz_k[k] = v;
    S->idx_off[k] = tot;
    tot += v;
  }
  DevBuf offs;
  if ((rc = offs.reserve(sizeof(int64_t) * count))) return cleanup(rc);
  e = cudaMalloc(&S->indices, sizeof(int32_t) * (tot > 0 ? tot : 1));
  if (e == cudaSuccess) e = cudaMemcpyAsync(offs.ptr, S->idx_off.data(), sizeof(int64_t) * count, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) { offs.release(); return cleanup(cuda_fail(e, "cudaMalloc(sample indices)")); }
  k_induce_fill<<<grid, 256, 0, st>>>(p->indptr, p->indices, (const uint32_t*)bitmaps.ptr, words,
                                      (const int32_t*)wordpre.ptr, S->nodes, (const int32_t*)nv.ptr, count, n,
                                      S->indptr, (const int64_t*)offs.ptr, S->indices);
  count_launch(c);
  e = cudaStreamSynchronize(st);
  offs.release();
  bitmaps.release(); vs.release(); nv.release(); wordpre.release();
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

GSG_API int gsg_sample_free(gsg_sample_t s) {
  if (!s) return GSG_OK;
  DeviceGuard dg(s->device);
  cudaFree(s->nodes);
  cudaFree(s->indptr);
  cudaFree(s->indices);
  delete s;
  return GSG_OK;
}

}  // extern "C"
