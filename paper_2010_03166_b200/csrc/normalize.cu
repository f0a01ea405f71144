// normalize.cu -- SURVEY §8(a) row a1: build Â (self loops, values), its transposed values
// (device gather form of Alg. 4) and the degree bins used by the SpMMs.
// Everything is stream-ordered; no host synchronization.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace gsg {
namespace {

__device__ __forceinline__ int bucket_of(int d) { return d <= 0 ? 0 : 32 - __clz(d); }

__global__ void k_zero(int32_t* __restrict__ p, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0;
}

// One warp per row: rowptr[i] = indptr[i] + self*i, the degree-bucket histogram and max
// degree, the per-row value of the degree modes (rowval[i] = fp32(1/(d_i+1)) row-self or
// fp32(1/d_i) row, reused by k_fill for Â_ij and, gathered at column j, for Âᵀ_ij = Â_ji),
// the row id of every raw entry (for k_fill) and -- self modes -- the self loop itself, placed
// after the row's neighbors below i (a 32-way warp search of the ascending list: a 1.3K-degree
// row needs 3 probe rounds; the id stores carry no loads).
__global__ void k_rows(int n, const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, int self,
                       int mode, int32_t* __restrict__ rowptr, float* __restrict__ rowval,
                       int32_t* __restrict__ counters, int32_t* __restrict__ rowid, int32_t* __restrict__ col,
                       float* __restrict__ val, float* __restrict__ valT) {
  __shared__ int hist[kBins];
  __shared__ int mx;
  if (threadIdx.x < kBins) hist[threadIdx.x] = 0;
  if (threadIdx.x == 0) mx = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0) rowptr[n] = (int32_t)(indptr[n] + (self ? n : 0));
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const int64_t b = indptr[i], e = indptr[i + 1];
    const int d0 = (int)(e - b);
    for (int64_t k = b + lane; k < e; k += 32) rowid[k] = i;  // stores only
    int64_t lo = b, hi = e;  // self-loop position: first entry > i, by a 32-way warp search
    while (self && lo < hi) {
      const int64_t step = (hi - lo + 31) >> 5;
      const int64_t pl = lo + lane * step;
      const unsigned m = __ballot_sync(0xffffffffu, pl < hi && __ldg(indices + pl) > i);
      if (m) {
        const int f = __ffs(m) - 1;
        hi = lo + f * step;
        lo = f ? lo + (int64_t)(f - 1) * step + 1 : hi;
      } else {  // every probe <= i: continue after the last probe below hi
        lo += ((hi - 1 - lo) / step) * step + 1;
      }
    }
    const int below = (int)(lo - b);  // neighbors with id < i
    if (lane == 0) {
      const int32_t o = (int32_t)(b + (self ? i : 0));
      rowptr[i] = o;
      const int d = d0 + self;
      atomicAdd(&hist[bucket_of(d)], 1);
      atomicMax(&mx, d);
      if (mode == GSG_NORM_ROW_SELF) rowval[i] = (float)(1.0 / ((double)d0 + 1.0));
      else if (mode == GSG_NORM_ROW) rowval[i] = d0 > 0 ? (float)(1.0 / (double)d0) : 0.f;
      if (self) {  // Â_ii = 1/(d_i+1) (row-self; sym: 1/sqrt((d_i+1)^2))
        col[o + below] = i;
        val[o + below] = valT[o + below] = (float)(1.0 / ((double)d0 + 1.0));
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < kBins && hist[threadIdx.x]) atomicAdd(&counters[threadIdx.x], hist[threadIdx.x]);
  if (threadIdx.x == 0) atomicMax(&counters[kBins + 1], mx);
}

// Edge-parallel fill: every raw entry k of row r goes to its slot of Â, shifted by one past the
// row's self loop: rowptr[r] + (k - indptr[r]) + [j > r], i.e. k + r + [j > r] in the self
// modes (rowptr[r] = indptr[r] + r) and k otherwise -- no per-row serialization (a warp-per-row
// loop spent ~45 us on the 1.3K-degree hub rows of config 5). Values of the requested
// normalization are computed in fp64 and rounded once to fp32. k_rows writes the self loops.
//
// For the degree-based modes the transposed value is a closed form of the column's degree
// (Âᵀ_ij = Â_ji: 1/(d_j+1) row-self, 1/d_j row, val itself for the symmetric mode), written
// here in the same fp64 -> fp32 rounding as Â_ji, so valT is bit-for-bit the permutation of
// val that Alg. 4 produces. GSG_NORM_VALUES needs the search (k_transpose_vals).
__global__ void k_fill(int64_t nnz, const int64_t* __restrict__ nnz_dev, const int64_t* __restrict__ indptr,
                       const int32_t* __restrict__ indices, const float* __restrict__ values, int mode,
                       const int32_t* __restrict__ rowid, const float* __restrict__ rowval, int32_t* __restrict__ col,
                       float* __restrict__ val, float* __restrict__ valT) {
  if (nnz_dev) nnz = *nnz_dev;  // device-sized subgraph: the entry count is indptr[n]
  const int self = (mode == GSG_NORM_ROW_SELF || mode == GSG_NORM_SYM_SELF);
  const bool by_row = (mode == GSG_NORM_ROW_SELF || mode == GSG_NORM_ROW);
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += T) {
    const int r = __ldg(rowid + k), c = __ldg(indices + k);
    const int64_t pos = self ? k + r + (c > r ? 1 : 0) : k;
    col[pos] = c;
    if (by_row) {                          // Â_rc = rowval[r], Âᵀ_rc = Â_cr = rowval[c]
      val[pos] = __ldg(rowval + r);
      valT[pos] = __ldg(rowval + c);
    } else if (mode == GSG_NORM_SYM_SELF) {
      const double dr = (double)(__ldg(indptr + r + 1) - __ldg(indptr + r));
      const double dc = (double)(__ldg(indptr + c + 1) - __ldg(indptr + c));
      val[pos] = valT[pos] = (float)(1.0 / sqrt((dr + 1.0) * (dc + 1.0)));
    } else {
      val[pos] = values[k];                // GSG_NORM_VALUES: valT by k_transpose_vals
    }
  }
}

// valT at slot (u, v) = val at slot (v, u): binary search for u in row v's ascending list.
// One warp per row u. This reproduces Alg. 4's DataTrans exactly (same structure, a pure
// permutation of val).
__global__ void k_transpose_vals(int n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                 const float* __restrict__ val, float* __restrict__ valT, int32_t* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
    const int b = rowptr[u], e = rowptr[u + 1];
    for (int k = b + lane; k < e; k += 32) {
      const int v = col[k];
      int lo = rowptr[v], hi = rowptr[v + 1] - 1;
      int found = -1;
      while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        const int c = col[mid];
        if (c == u) { found = mid; break; }
        if (c < u) lo = mid + 1; else hi = mid - 1;
      }
      if (found < 0) { atomicExch(err, 1); valT[k] = __int_as_float(0x7fc00000); }
      else valT[k] = val[found];
    }
  }
}

// Rows by DESCENDING degree bucket. Every block derives the bucket offsets from the finished
// histogram itself (exclusive sums in descending bucket order; n_heavy = rows with
// deg' >= kHeavyMinDeg), then ranks its rows in shared memory and reserves each bucket's range
// with one global atomic per (block, bucket) on a zeroed cursor (the order within a bucket is
// immaterial: every row is summed by one warp or CTA in CSR order).
__global__ void k_bin_scatter(int n, const int32_t* __restrict__ rowptr, int32_t* __restrict__ counters,
                              int32_t* __restrict__ perm, int4* __restrict__ htask, int32_t* __restrict__ hcount,
                              int hseg_len) {
  __shared__ int cnt[kBins], base[kBins], off[kBins];
  if (threadIdx.x == 0) {
    int acc = 0, heavy = 0, mega = 0;
    const int hb = 32 - __clz(kHeavyMinDeg), mb = 32 - __clz(kMegaMinDeg);
    for (int b = kBins - 1; b >= 0; b--) {
      off[b] = acc;
      acc += counters[b];
      if (b >= hb) heavy += counters[b];
      if (b >= mb) mega += counters[b];
    }
    if (blockIdx.x == 0) {
      counters[kBins] = heavy;
      counters[kNMega] = mega;  // rows with deg' >= kMegaMinDeg lead perm
    }
  }
  __syncthreads();
  for (int i0 = blockIdx.x * blockDim.x; i0 < n; i0 += gridDim.x * blockDim.x) {
    if (threadIdx.x < kBins) cnt[threadIdx.x] = 0;
    __syncthreads();
    const int i = i0 + threadIdx.x;
    int b = -1, r = 0;
    if (i < n) {
      const int rb = rowptr[i], d = rowptr[i + 1] - rb;
      b = bucket_of(d);
      r = atomicAdd(&cnt[b], 1);
      if (htask && d >= kHeavyMinDeg) {
        // the heavy row's warp segments for the SpMM: ceil(d / kHSeg) equal pieces, contiguous
        // in htask at a place reserved by one atomic (the order of rows in the list is
        // immaterial: each row's partial sums are combined in segment order)
        const int sc = (d + hseg_len - 1) / hseg_len, len = (d + sc - 1) / sc;
        const int first = atomicAdd(&counters[kNHSeg], sc);
        hcount[first] = sc;
        for (int s2 = 0; s2 < sc; s2++) htask[first + s2] = make_int4(i, rb + s2 * len, min(rb + d, rb + (s2 + 1) * len), first);
      }
    }
    __syncthreads();
    if (threadIdx.x < kBins && cnt[threadIdx.x])
      base[threadIdx.x] = off[threadIdx.x] + atomicAdd(&counters[kBins + 2 + threadIdx.x], cnt[threadIdx.x]);
    __syncthreads();
    if (b >= 0) perm[base[b] + r] = i;
    __syncthreads();
  }
}

// Segment length of heavy rows: about the neighbors one warp of the SpMM's persistent grid gathers
// per launch (nnz' / (SMs x 24 warps)), in [160, kHSeg], a multiple of 32. On a small subgraph the
// few tasks per warp make the longest task set the kernel's length, so finer segments balance
// it; on a large one they only add combine work (SpMM steps, GSG_HSEG_LEN=160 / 192 / 224 / 256:
// config 3 0.542 / 0.556 / 0.565 / 0.575 ms, config 4 2.062 / 1.952 / 1.960 / 1.968, config 5
// 2.887 / 2.898 / 2.887 / 2.888; profiles/r02_hseg_len_ab.txt). GSG_HSEG_LEN fixes it (A/B).
int hseg_len(const gsg_ctx* ctx, int64_t nnz_hat) {
  static const int env = getenv("GSG_HSEG_LEN") ? atoi(getenv("GSG_HSEG_LEN")) : 0;
  if (env >= 32) return env;
  // 16 warps per SM: the f <= 512 launches run two 8-warp CTAs/SM since the dynamic schedule, and
  // with claimed tasks longer segments cost less than the combines they save (config 4 192 -> 256:
  // 1.903 -> 1.874 ms; config 3 stays within 0.3 % at 192; profiles/r02_hseg_len_ab.txt)
  const int64_t per_warp = nnz_hat / ((int64_t)ctx->num_sms * 16);
  const int64_t v = (per_warp + 31) / 32 * 32;  // rounded up to whole 32-neighbor groups
  return (int)std::min<int64_t>(kHSeg, std::max<int64_t>(160, v));
}

}  // namespace

int normalize_launch(gsg_ctx* ctx, gsg_subgraph* sg, int mode) {
  GSG_CHECK(mode >= GSG_NORM_ROW_SELF && mode <= GSG_NORM_VALUES, GSG_EINVAL, "bad norm_mode %d", mode);
  GSG_CHECK(mode != GSG_NORM_VALUES || sg->has_values, GSG_EINVAL, "GSG_NORM_VALUES needs uploaded edge values");
  const int self = (mode == GSG_NORM_ROW_SELF || mode == GSG_NORM_SYM_SELF);
  const int64_t nh = sg->nnz + (self ? sg->n : 0);
  GSG_CHECK(nh < (int64_t)INT32_MAX, GSG_EUNSUPPORTED, "nnz_hat %lld exceeds int32", (long long)nh);
  const int n = sg->n;
  cudaStream_t st = ctx->stream;
  if ((size_t)nh > sg->cap_hat) {
    cudaFree(sg->col); cudaFree(sg->val); cudaFree(sg->valT); cudaFree(sg->rowid);
    sg->col = sg->rowid = nullptr; sg->val = sg->valT = nullptr;
    size_t c = (size_t)(nh > 0 ? nh : 1);
    GSG_CUDA(cudaMalloc(&sg->col, c * sizeof(int32_t)));
    GSG_CUDA(cudaMalloc(&sg->val, c * sizeof(float)));
    GSG_CUDA(cudaMalloc(&sg->valT, c * sizeof(float)));
    GSG_CUDA(cudaMalloc(&sg->rowid, c * sizeof(int32_t)));
    sg->cap_hat = c;
  }
  sg->nnz_hat = nh;
  sg->norm_mode = mode;
  const int hl = hseg_len(ctx, nh);
  {  // heavy-row segments: sum over heavy rows of ceil(deg'/hl) <= nnz'/hl + nnz'/kHeavyMinDeg
    const size_t cap = (size_t)(nh / hl + nh / kHeavyMinDeg + 1);
    if (cap > sg->cap_hseg) {
      cudaFree(sg->htask); cudaFree(sg->hcount);
      sg->htask = nullptr; sg->hcount = nullptr;
      GSG_CUDA(cudaMalloc(&sg->htask, sizeof(int4) * cap));
      GSG_CUDA(cudaMalloc(&sg->hcount, sizeof(int32_t) * cap));
      sg->cap_hseg = cap;
    }
  }
  ProfScope ps(ctx, GSG_K_NORM, 16.0 * nh + 24.0 * n, 0.0);
  // counters zeroed by a kernel, not a memset node: inside the step's CUDA graph a memset
  // node cost ~7.5 us of idle time before the next kernel (r02 timeline), a kernel < 1 us
  k_zero<<<1, 128, 0, st>>>(sg->counters, 3 * kBins + 8);
  count_launch(ctx);
  const int T = 256;
  int grid = (n + 1 + T - 1) / T;
  if (grid > ctx->num_sms * 8) grid = ctx->num_sms * 8;
  if (grid < 1) grid = 1;
  int wgrid = (int)(((int64_t)n * 32 + T - 1) / T);
  if (wgrid > ctx->num_sms * 16) wgrid = ctx->num_sms * 16;
  if (wgrid < 1) wgrid = 1;
  k_rows<<<wgrid, T, 0, st>>>(n, sg->indptr, sg->indices, self, mode, sg->rowptr, sg->rowval, sg->counters, sg->rowid,
                               sg->col, sg->val, sg->valT);
  count_launch(ctx);
  if (n > 0) {
    if (sg->nnz > 0) {
      int64_t eg = (sg->nnz + T - 1) / T;
      if (eg > (int64_t)ctx->num_sms * 16) eg = (int64_t)ctx->num_sms * 16;
      k_fill<<<(int)eg, T, 0, st>>>(sg->nnz, sg->dev_sized ? sg->indptr + n : nullptr, sg->indptr, sg->indices,
                                    sg->has_values ? sg->values : nullptr, mode, sg->rowid, sg->rowval, sg->col,
                                    sg->val, sg->valT);
      count_launch(ctx);
    }
    if (mode == GSG_NORM_VALUES) {
      k_transpose_vals<<<wgrid, T, 0, st>>>(n, sg->rowptr, sg->col, sg->val, sg->valT, sg->counters + 3 * kBins + 4);
      count_launch(ctx);
    }
    k_bin_scatter<<<grid, T, 0, st>>>(n, sg->rowptr, sg->counters, sg->perm, sg->htask, sg->hcount, hl);
    count_launch(ctx);
  }
  GSG_CUDA(cudaGetLastError());
  return GSG_OK;
}

}  // namespace gsg
