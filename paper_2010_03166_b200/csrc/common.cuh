// common.cuh -- shared internals of libgsg.so (context, subgraph, error plumbing).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "gsg.h"

namespace gsg {

constexpr int kHeavyMinDeg = 256;   // deg' >= this -> CTA-cooperative row (degree bin "heavy")
constexpr int kMegaMinDeg = 2048;   // deg' >= this -> the row is split over kMegaSegs CTAs ("mega")
constexpr int kMegaSegs = 8;
constexpr int kBins = 32;           // log2 degree buckets
constexpr int kNMega = 3 * kBins + 6;  // counters[]: number of mega rows (the first ones in perm)
constexpr int kHSeg = 256;          // heavy rows are cut into warp segments of <= kHSeg neighbors (normalize: 160-256 by size)
constexpr int kNHSeg = 3 * kBins + 7;  // counters[]: number of heavy-row segments (normalize)

void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

#define GSG_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return ::gsg::cuda_fail(_e, #call); \
  } while (0)

#define GSG_CHECK(cond, code, ...)                       \
  do {                                                   \
    if (!(cond)) return ::gsg::fail(code, __VA_ARGS__);  \
  } while (0)

// Makes `dev` current for the scope of an API call and restores the caller's device after.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// NVTX range around a public entry point (header-only NVTX3: a no-op unless a tool such as
// Nsight Systems injects itself), named by the SURVEY §8(a) row it implements.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Grow-only device buffer.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int reserve(size_t b) {
    if (b <= bytes) return GSG_OK;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    size_t nb = b + b / 4 + 256;
    cudaError_t e = cudaMalloc(&ptr, nb);
    if (e != cudaSuccess) { ptr = nullptr; return fail(GSG_ENOMEM, "cudaMalloc(%zu) failed: %s", nb, cudaGetErrorString(e)); }
    bytes = nb;
    return GSG_OK;
  }
  void release() { if (ptr) cudaFree(ptr); ptr = nullptr; bytes = 0; }
};

}  // namespace gsg

namespace gsg {
// Per-class CUDA-event profiler (gsg_ctx_profile).
struct Profiler {
  bool on = false;
  struct Rec { int cls, row, pending; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> free_ev;
  double bytes[GSG_K_CLASSES] = {}, flops[GSG_K_CLASSES] = {};
  cudaEvent_t get() {
    if (!free_ev.empty()) { cudaEvent_t e = free_ev.back(); free_ev.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};
}  // namespace gsg

struct gsg_sample;

struct gsg_ctx {
  gsg::Profiler prof;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  int64_t launches = 0;
  int prof_row = -1;       // SURVEY §8(a) row of the launches being issued (GSG_K_A*), -1 = none
  gsg::DevBuf ws_splitk;   // split-K partials (context stream)
  gsg::DevBuf ws_splitk_side;  // split-K partials of the GEMMs that may be forked onto the side stream
  bool side_ws = false;        // gemm_launch uses ws_splitk_side (set around those GEMMs, forked or not)
  gsg::DevBuf ws_T;        // T = dZ Wᵀ (fp32)
  gsg::DevBuf ws_dZ;       // masked dZ (fp32)
  gsg::DevBuf ws_lp0;      // bf16 scratch (W copy)
  gsg::DevBuf ws_lp1;      // bf16 scratch (dZ copy / T copy)
  gsg::DevBuf ws_lp2;      // bf16 scratch
  gsg::DevBuf ws_loss;     // per-block loss partials
  gsg::DevBuf ws_x3[2];    // GSG_PREC_FP32X3 split operand copies (A3, B3), context stream
  gsg::DevBuf ws_x3_side[2];  // the same for the GEMMs that may be forked onto the side stream
  gsg::DevBuf ws_x3dz;     // FP32X3: dZ's (dS's) lo, split once per layer backward (head) for both of its GEMMs
  gsg::DevBuf ws_x3hl;     // FP32X3: H_L's lo, split once per head call for S and dW_mlp
  gsg::DevBuf ws_hseg;     // SpMM heavy-row segment partials
  gsg::DevBuf ws_hsegctr;  // SpMM heavy-row (row, chunk) arrival counters, zero between launches
  gsg::DevBuf ws_mega;     // SpMM mega-row segment partials
  gsg::DevBuf ws_megactr;  // SpMM mega-row (row, chunk) arrival counters, zero between launches
  gsg::DevBuf ws_taskctr;  // SpMM dynamic warp-task counter + CTA exit counter, zero between launches
  cudaStream_t side = nullptr;       // fork/join side stream (layer backward: dW next to T -> dX)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // gsg_frontier_sample: scratch of a call (V_s bitmaps, insertion lists, sizes) and the device
  // arrays of freed sample batches kept for the next call -- a config-5 batch of 888 holds
  // 8.3 GB of induced indices, and allocating / freeing that per call cost 2-500 ms of host time
  gsg::DevBuf ws_sbits, ws_svs, ws_snv, ws_swordpre, ws_snnz;
  std::vector<std::pair<void*, size_t>> spare;  // device buffers of freed samples (ptr, bytes)
  std::vector<gsg_sample*> live_samples;        // samples whose buffers return to `spare` when freed
};

struct gsg_subgraph {
  int device = 0;
  int32_t n = 0;
  int64_t nnz = 0;          // raw entries (no self loops)
  int64_t nnz_hat = 0;      // entries of Â (after normalization)
  int norm_mode = -1;
  int32_t host_max_deg = -1;
  int32_t cap_n = 0;        // allocated capacity (gsg_subgraph_assign reuses arrays)
  int64_t cap_nnz = 0;
  bool has_values = false;
  bool dev_sized = false;   // gsg_subgraph_create_device: n is fixed, the entry count lives on the
                            // device (indptr[n]); host nnz / nnz_hat are capacities
  // raw structure (device)
  int64_t* indptr = nullptr;    // [n+1]
  int32_t* indices = nullptr;   // [nnz]
  float* values = nullptr;      // [nnz] or null
  // normalized Â (device)
  int32_t* rowptr = nullptr;    // [n+1]
  int32_t* col = nullptr;       // [nnz_hat]
  float* val = nullptr;         // [nnz_hat]
  float* valT = nullptr;        // [nnz_hat]
  int32_t* perm = nullptr;      // [n] rows by descending degree bucket
  int32_t* rowid = nullptr;     // [nnz] row of each raw entry (normalize scratch)
  float* rowval = nullptr;      // [n] per-row value of the degree modes (1/(d+1) or 1/d), fp64-rounded
  int32_t* counters = nullptr;  // [kBins + 8]: bucket counts ..., [kBins]=n_heavy, [kBins+1]=max_deg
  int4* htask = nullptr;        // [segments] heavy-row warp segments: (row, k_begin, k_end, first segment of the row)
  int32_t* hcount = nullptr;    // [segments] at a row's first segment: its number of segments
  size_t cap_hseg = 0;
  size_t cap_hat = 0;
};

namespace gsg {
inline void count_launch(gsg_ctx* c, int k = 1) { c->launches += k; }

// Brackets the kernels of one API-level launch with events when profiling is on.
struct ProfScope {
  gsg_ctx* c;
  int cls;
  cudaEvent_t a = nullptr;
  ProfScope(gsg_ctx* c_, int cls_, double bytes, double flops) : c(c_), cls(cls_) {
    if (!c->prof.on) return;
    c->prof.bytes[cls] += bytes;
    c->prof.flops[cls] += flops;
    if (c->prof_row >= 0) {
      c->prof.bytes[c->prof_row] += bytes;
      c->prof.flops[c->prof_row] += flops;
    }
    a = c->prof.get();
    record(a);
  }
  // inside a stream capture, external records stay timing events of the replayed graph
  void record(cudaEvent_t e) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(c->stream, &st);
    if (st == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, c->stream, cudaEventRecordExternal);
    else cudaEventRecord(e, c->stream);
  }
  ~ProfScope() {
    if (!a) return;
    cudaEvent_t b = c->prof.get();
    record(b);
    c->prof.recs.push_back({cls, c->prof_row, c->prof_row >= 0 ? 2 : 1, a, b});
  }
};

// Tags the launches issued in its scope with a SURVEY §8(a) row (GSG_K_A*).
struct RowTag {
  gsg_ctx* c;
  int prev;
  RowTag(gsg_ctx* c_, int row) : c(c_), prev(c_->prof_row) { c->prof_row = row; }
  ~RowTag() { c->prof_row = prev; }
};

// launch wrappers implemented in the .cu files
int normalize_launch(gsg_ctx* ctx, gsg_subgraph* sg, int mode);
// ReLU bitmasks (gsg.h "ReLU bitmask"): `out` receives 1[result > 0] of a ReLU epilogue, `in`
// replaces the fp32 gate operand of a ReLU' (mask) epilogue. Strides in 32-bit words.
struct BitsIO {
  uint32_t* out = nullptr;
  int64_t ldo = 0;
  const uint32_t* in = nullptr;
  int64_t ldi = 0;
};
int spmm_launch(gsg_ctx* ctx, const gsg_subgraph* sg, int transpose, int f, const float* X, int64_t ldx,
                float* Y, int64_t ldy, void* Ylp, int64_t ldylp, const float* mask, int64_t ldm, int relu = 0,
                int accum = 0, const BitsIO& bits = BitsIO{});
// FP32X3 lo operands the caller already computed (split_lo_launch of the same stored matrix),
// e.g. dZ's, shared by the backward's T and dW GEMMs; nullptr = split inside the GEMM call.
struct X3Lo {
  const float* a = nullptr;
  int64_t lda = 0;
  const float* b = nullptr;
  int64_t ldb = 0;
};
int gemm_launch(gsg_ctx* ctx, int M, int N, int K, const void* A, int64_t lda, int transA,
                const void* B, int64_t ldb, int transB, float* C, int64_t ldc, void* Clp, int64_t ldclp,
                int precision, int epilogue, const float* aux, int64_t ldaux, int split_k, int accumulate,
                const BitsIO& bits = BitsIO{}, const X3Lo& pre = X3Lo{});
// lo = x - trunc_tf32(x) of a row-major fp32 matrix (FP32X3 operand split), ldd % 4 == 0
int split_lo_launch(gsg_ctx* ctx, int rows, int cols, const float* src, int64_t lds, float* dst, int64_t ldd);
bool x3_implicit();  // FP32X3 runs the implicit-hi path (GSG_X3_IMPLICIT, default 1)
int to_bf16_launch(gsg_ctx* ctx, int rows, int cols, const float* src, int64_t lds, void* dst, int64_t ldd);
int gather_rows_launch(gsg_ctx* ctx, int rows, int64_t row_bytes, const void* src, int64_t src_pitch,
                       const int32_t* idx, void* dst, int64_t dst_pitch);
int mask_launch(gsg_ctx* ctx, int rows, int cols, const float* dH, int64_t lddh, const float* H, int64_t ldh,
                float* dZ, int64_t lddz, void* dZlp, int64_t lddzlp);
int mask_bits_launch(gsg_ctx* ctx, int rows, int cols, const float* dH, int64_t lddh, const uint32_t* bits,
                     int64_t ldb, float* dZ, int64_t lddz, void* dZlp, int64_t lddzlp);
int head_loss_launch(gsg_ctx* ctx, int n, int C, int kind, const float* S, int64_t lds, const void* labels,
                     const float* node_w, float* dS, float* loss);
void sampler_detach(gsg_ctx* ctx);  // gsg_ctx_destroy: live samples stop returning buffers to it
}  // namespace gsg
