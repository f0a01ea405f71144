// api.cu -- the C ABI of libgsg.so (include/gsg.h): argument checking, ownership, and the
// composition of the hot-path kernels into the paper's per-layer calls.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstdarg>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"

namespace gsg {

static thread_local char g_err[2048] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(e == cudaErrorMemoryAllocation ? GSG_ENOMEM : GSG_ECUDA, "%s: %s (%s)", what, cudaGetErrorString(e),
              cudaGetErrorName(e));
}

}  // namespace gsg

using namespace gsg;

namespace {

int check_ctx(gsg_ctx_t c) { return c ? GSG_OK : fail(GSG_EINVAL, "NULL context"); }

// ---- host-side CSR validation (gsg.h: gsg_subgraph_upload) ----
int validate_csr(int32_t n, int64_t nnz, const int64_t* ip, const int32_t* ix) {
  if (ip[0] != 0) return fail(GSG_EGRAPH, "indptr[0] = %lld, expected 0", (long long)ip[0]);
  for (int32_t i = 0; i < n; i++)
    if (ip[i + 1] < ip[i]) return fail(GSG_EGRAPH, "indptr decreases at row %d", i);
  if (ip[n] != nnz) return fail(GSG_EGRAPH, "indptr[n] = %lld != nnz = %lld", (long long)ip[n], (long long)nnz);
  for (int32_t i = 0; i < n; i++) {
    for (int64_t k = ip[i]; k < ip[i + 1]; k++) {
      const int32_t j = ix[k];
      if (j < 0 || j >= n) return fail(GSG_EGRAPH, "edge (%d, %d): index out of range [0, %d)", i, j, n);
      if (j == i) return fail(GSG_EGRAPH, "edge (%d, %d): self loop (normalization adds it)", i, j);
      if (k > ip[i] && ix[k - 1] >= j)
        return fail(GSG_EGRAPH, "edge (%d, %d): row %d not strictly ascending (previous %d)", i, j, i, ix[k - 1]);
    }
  }
  for (int32_t i = 0; i < n; i++) {
    for (int64_t k = ip[i]; k < ip[i + 1]; k++) {
      const int32_t j = ix[k];
      int64_t lo = ip[j], hi = ip[j + 1] - 1;
      bool found = false;
      while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (ix[mid] == i) { found = true; break; }
        if (ix[mid] < i) lo = mid + 1; else hi = mid - 1;
      }
      if (!found) return fail(GSG_EGRAPH, "edge (%d, %d) has no reverse edge (%d, %d): not symmetric", i, j, j, i);
    }
  }
  return GSG_OK;
}

int alloc_subgraph(gsg_ctx* ctx, int32_t n, int64_t nnz, bool has_values, gsg_subgraph** out) {
  GSG_CHECK(n >= 0 && nnz >= 0, GSG_EINVAL, "negative n or nnz");
  GSG_CHECK(nnz + (int64_t)n < (int64_t)INT32_MAX, GSG_EUNSUPPORTED, "nnz + n exceeds int32 indexing");
  auto* sg = new gsg_subgraph;
  sg->device = ctx->device;
  sg->n = n;
  sg->nnz = nnz;
  sg->cap_n = n;
  sg->cap_nnz = nnz;
  sg->has_values = has_values;
  cudaError_t e = cudaSuccess;
  auto A = [&](void** p, size_t b) { if (e == cudaSuccess) e = cudaMalloc(p, b > 0 ? b : 16); };
  A((void**)&sg->indptr, sizeof(int64_t) * (n + 1));
  A((void**)&sg->indices, sizeof(int32_t) * nnz);
  if (has_values) A((void**)&sg->values, sizeof(float) * nnz);
  A((void**)&sg->rowptr, sizeof(int32_t) * (n + 1));
  A((void**)&sg->perm, sizeof(int32_t) * n);
  A((void**)&sg->rowval, sizeof(float) * n);
  A((void**)&sg->counters, sizeof(int32_t) * (3 * kBins + 8));
  if (e != cudaSuccess) {
    gsg_subgraph_free(sg);
    return cuda_fail(e, "cudaMalloc(subgraph)");
  }
  *out = sg;
  return GSG_OK;
}

// ---- NCCL (resolved at run time) ----
struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  bool ok = false;
};

Nccl load_nccl() {
  Nccl N;
  {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      N.GetUniqueId = (decltype(N.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      N.CommInitRank = (decltype(N.CommInitRank))dlsym(h, "ncclCommInitRank");
      N.CommDestroy = (decltype(N.CommDestroy))dlsym(h, "ncclCommDestroy");
      N.AllReduce = (decltype(N.AllReduce))dlsym(h, "ncclAllReduce");
      N.GroupStart = (decltype(N.GroupStart))dlsym(h, "ncclGroupStart");
      N.GroupEnd = (decltype(N.GroupEnd))dlsym(h, "ncclGroupEnd");
      N.GetErrorString = (decltype(N.GetErrorString))dlsym(h, "ncclGetErrorString");
      N.CommGetAsyncError = (decltype(N.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
      N.CommAbort = (decltype(N.CommAbort))dlsym(h, "ncclCommAbort");
      N.ok = N.GetUniqueId && N.CommInitRank && N.CommDestroy && N.AllReduce && N.GroupStart && N.GroupEnd &&
             N.GetErrorString && N.CommGetAsyncError && N.CommAbort;
    }
  }
  return N;
}

Nccl& nccl() {
  static Nccl N = load_nccl();  // resolved once, thread-safe (function-local static initialization)
  return N;
}

int nccl_fail(ncclResult_t r, const char* what) {
  return fail(GSG_ENCCL, "%s: %s", what, nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error");
}

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Fork / join of the context's side stream for a GEMM that only shares read-only inputs with
// the work that follows it on the context stream: the constructor forks (the side stream waits
// for everything enqueued so far) and redirects launches to the side stream, back() returns
// them to the context stream, and the destructor joins -- on every exit path, so an error can
// never leave an unjoined stream inside a graph capture.
struct SideFork {
  gsg_ctx* c;
  cudaStream_t main;
  bool on, away = false;
  SideFork(gsg_ctx* c_, bool on_) : c(c_), main(c_->stream), on(on_) {
    if (!on) return;
    cudaEventRecord(c->ev_fork, main);
    cudaStreamWaitEvent(c->side, c->ev_fork, 0);
    c->stream = c->side;
    away = true;
  }
  void back() {
    if (!away) return;
    cudaEventRecord(c->ev_join, c->side);
    c->stream = main;
    away = false;
  }
  ~SideFork() {
    if (!on) return;
    back();
    cudaStreamWaitEvent(main, c->ev_join, 0);
  }
};

bool fork_enabled() {
  static const bool f = !(getenv("GSG_BWD_FORK") && atoi(getenv("GSG_BWD_FORK")) == 0);
  return f;
}

// GSG_BWD_TFIRST (A/B): 0 dW first (default), 1 T first in every layer, 2 T first where the
// layer's input is narrower than its output (layer 1); GSG_HEAD_DHFIRST=1: the head's dH_L
// before its forked dW_mlp
bool t_first(int f_in, int f_out) {
  static const int m = getenv("GSG_BWD_TFIRST") ? atoi(getenv("GSG_BWD_TFIRST")) : 0;
  return m == 1 || (m == 2 && f_in < f_out);
}
bool head_dh_first() {
  static const bool f = getenv("GSG_HEAD_DHFIRST") && atoi(getenv("GSG_HEAD_DHFIRST")) == 1;
  return f;
}

// The bf16 weight operand of a layer GEMM: the caller's own copy (GSG_W_BF16: W is bf16 with
// ldw in bf16 elements) or a conversion into the context workspace.
int bf16_weight(gsg_ctx* c, const float* W, int64_t ldw, int f_in, int f_out, int flags, const void** out,
                int64_t* ld_out) {
  if (flags & GSG_W_BF16) {
    GSG_CHECK(ldw >= f_out && ldw % 8 == 0 && (uintptr_t)W % 16 == 0, GSG_EINVAL,
              "GSG_W_BF16: bf16 W needs ldw >= f_out, ldw %% 8 == 0 and 16-byte alignment");
    *out = W;
    *ld_out = ldw;
    return GSG_OK;
  }
  const int64_t ldwl = round_up(f_out, 8);
  if (int rc = c->ws_lp0.reserve(sizeof(uint16_t) * f_in * ldwl)) return rc;
  if (int rc = to_bf16_launch(c, f_in, f_out, W, ldw, c->ws_lp0.ptr, ldwl)) return rc;
  *out = c->ws_lp0.ptr;
  *ld_out = ldwl;
  return GSG_OK;
}

}  // namespace

extern "C" {

GSG_API const char* gsg_last_error(void) { return g_err; }

GSG_API int gsg_ctx_create(int device, void* cuda_stream, gsg_ctx_t* out) {
  GSG_CHECK(out, GSG_EINVAL, "out is NULL");
  *out = nullptr;
  int count = 0;
  GSG_CUDA(cudaGetDeviceCount(&count));
  GSG_CHECK(device >= 0 && device < count, GSG_EINVAL, "device %d out of range (%d devices)", device, count);
  cudaDeviceProp prop;
  GSG_CUDA(cudaGetDeviceProperties(&prop, device));
  GSG_CHECK(prop.major == 10 && prop.minor == 0, GSG_EUNSUPPORTED,
            "device %d is sm_%d%d; libgsg is built for sm_100a (B200) only", device, prop.major, prop.minor);
  DeviceGuard dg(device);
  auto* c = new gsg_ctx;
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  c->stream = static_cast<cudaStream_t>(cuda_stream);
  GSG_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  GSG_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  GSG_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  *out = c;
  return GSG_OK;
}

GSG_API int gsg_ctx_destroy(gsg_ctx_t c) {
  if (!c) return GSG_OK;
  DeviceGuard dg(c->device);
  cudaStreamSynchronize(c->stream);
  c->ws_splitk.release(); c->ws_splitk_side.release(); c->ws_T.release(); c->ws_dZ.release();
  c->ws_lp0.release(); c->ws_lp1.release(); c->ws_lp2.release(); c->ws_loss.release();
  c->ws_mega.release(); c->ws_megactr.release(); c->ws_taskctr.release(); c->ws_hseg.release(); c->ws_hsegctr.release();
  for (int i = 0; i < 2; i++) { c->ws_x3[i].release(); c->ws_x3_side[i].release(); }
  c->ws_x3dz.release(); c->ws_x3hl.release();
  c->ws_sbits.release(); c->ws_svs.release(); c->ws_snv.release(); c->ws_swordpre.release(); c->ws_snnz.release();
  gsg::sampler_detach(c);  // live samples keep their arrays and free them themselves
  for (auto& b : c->spare) cudaFree(b.first);
  for (auto& r : c->prof.recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : c->prof.free_ev) cudaEventDestroy(e);
  if (c->side) { cudaStreamSynchronize(c->side); cudaStreamDestroy(c->side); }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  delete c;
  return GSG_OK;
}

GSG_API int gsg_ctx_set_stream(gsg_ctx_t c, void* s) {
  if (int rc = check_ctx(c)) return rc;
  c->stream = static_cast<cudaStream_t>(s);
  return GSG_OK;
}

GSG_API void* gsg_ctx_stream(gsg_ctx_t c) { return c ? (void*)c->stream : nullptr; }

GSG_API int gsg_ctx_sync(gsg_ctx_t c) {
  if (int rc = check_ctx(c)) return rc;
  DeviceGuard dg(c->device);
  GSG_CUDA(cudaStreamSynchronize(c->stream));
  GSG_CUDA(cudaGetLastError());
  return GSG_OK;
}

GSG_API int gsg_ctx_wait_event(gsg_ctx_t c, void* ev) {
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(ev, GSG_EINVAL, "NULL event");
  DeviceGuard dg(c->device);
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  GSG_CUDA(cudaStreamIsCapturing(c->stream, &st));
  GSG_CUDA(cudaStreamWaitEvent(c->stream, static_cast<cudaEvent_t>(ev),
                               st == cudaStreamCaptureStatusActive ? cudaEventWaitExternal : 0));
  return GSG_OK;
}

GSG_API int64_t gsg_ctx_launch_count(gsg_ctx_t c) { return c ? c->launches : -1; }

GSG_API int gsg_ctx_profile(gsg_ctx_t c, int enable) {
  if (int rc = check_ctx(c)) return rc;
  c->prof.on = enable != 0;
  return GSG_OK;
}

GSG_API int gsg_ctx_profile_read(gsg_ctx_t c, int kclass, double* total_ms, int64_t* launches, double* alg_bytes,
                                 double* alg_flops) {
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(kclass >= 0 && kclass < GSG_K_CLASSES, GSG_EINVAL, "bad kernel class %d", kclass);
  DeviceGuard dg(c->device);
  GSG_CUDA(cudaStreamSynchronize(c->stream));
  double ms = 0.0;
  int64_t cnt = 0;
  std::vector<gsg::Profiler::Rec> keep;
  for (auto& r : c->prof.recs) {
    if (r.cls != kclass && r.row != kclass) { keep.push_back(r); continue; }
    float t = 0.f;
    GSG_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    ms += t;
    cnt++;
    if (--r.pending > 0) {  // the record still owes its time to its other class
      if (r.cls == kclass) r.cls = -1; else r.row = -1;
      keep.push_back(r);
      continue;
    }
    c->prof.free_ev.push_back(r.a);
    c->prof.free_ev.push_back(r.b);
  }
  c->prof.recs.swap(keep);
  if (total_ms) *total_ms = ms;
  if (launches) *launches = cnt;
  if (alg_bytes) *alg_bytes = c->prof.bytes[kclass];
  if (alg_flops) *alg_flops = c->prof.flops[kclass];
  c->prof.bytes[kclass] = c->prof.flops[kclass] = 0.0;
  return GSG_OK;
}

// ------------------------------------------------------------------------------ subgraph
GSG_API int gsg_subgraph_upload(gsg_ctx_t c, int32_t n, int64_t nnz, const int64_t* h_indptr, const int32_t* h_indices,
                                const float* h_values, int validate, gsg_subgraph_t* out) {
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(out, GSG_EINVAL, "out is NULL");
  *out = nullptr;
  GSG_CHECK(n >= 0 && nnz >= 0, GSG_EINVAL, "negative n (%d) or nnz (%lld)", n, (long long)nnz);
  GSG_CHECK(h_indptr && (nnz == 0 || h_indices), GSG_EINVAL, "NULL indptr/indices");
  if (validate) {
    if (int rc = validate_csr(n, nnz, h_indptr, h_indices)) return rc;
  } else {
    GSG_CHECK(h_indptr[n] == nnz, GSG_EGRAPH, "indptr[n] = %lld != nnz = %lld", (long long)h_indptr[n], (long long)nnz);
  }
  DeviceGuard dg(c->device);
  gsg_subgraph* sg = nullptr;
  if (int rc = alloc_subgraph(c, n, nnz, h_values != nullptr, &sg)) return rc;
  int32_t mx = 0;
  for (int32_t i = 0; i < n; i++) mx = (int32_t)std::max<int64_t>(mx, h_indptr[i + 1] - h_indptr[i]);
  sg->host_max_deg = mx;
  cudaError_t e = cudaMemcpyAsync(sg->indptr, h_indptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess && nnz)
    e = cudaMemcpyAsync(sg->indices, h_indices, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess && h_values && nnz)
    e = cudaMemcpyAsync(sg->values, h_values, sizeof(float) * nnz, cudaMemcpyHostToDevice, c->stream);
  if (e != cudaSuccess) { gsg_subgraph_free(sg); return cuda_fail(e, "cudaMemcpyAsync(upload)"); }
  *out = sg;
  return GSG_OK;
}

GSG_API int gsg_subgraph_assign(gsg_ctx_t c, gsg_subgraph_t sg, int32_t n, int64_t nnz, const int64_t* h_indptr,
                                const int32_t* h_indices, const float* h_values, int validate) {
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(sg, GSG_EINVAL, "NULL subgraph");
  GSG_CHECK(n >= 0 && nnz >= 0, GSG_EINVAL, "negative n (%d) or nnz (%lld)", n, (long long)nnz);
  GSG_CHECK(h_indptr && (nnz == 0 || h_indices), GSG_EINVAL, "NULL indptr/indices");
  GSG_CHECK(nnz + (int64_t)n < (int64_t)INT32_MAX, GSG_EUNSUPPORTED, "nnz + n exceeds int32 indexing");
  cudaPointerAttributes pa{};
  const bool on_device = cudaPointerGetAttributes(&pa, h_indptr) == cudaSuccess && pa.type == cudaMemoryTypeDevice;
  cudaGetLastError();  // clear a pointer-query error for plain (unregistered) host memory
  if (on_device) {
    GSG_CHECK(!validate, GSG_EINVAL, "validate needs host arrays (the CSR is device-resident)");
  } else if (validate) {
    if (int rc = validate_csr(n, nnz, h_indptr, h_indices)) return rc;
  } else {
    GSG_CHECK(h_indptr[n] == nnz, GSG_EGRAPH, "indptr[n] = %lld != nnz = %lld", (long long)h_indptr[n], (long long)nnz);
  }
  DeviceGuard dg(c->device);
  if (n > sg->cap_n) {
    cudaFree(sg->indptr); cudaFree(sg->rowptr); cudaFree(sg->perm); cudaFree(sg->rowval);
    sg->indptr = nullptr; sg->rowptr = sg->perm = nullptr; sg->rowval = nullptr;
    GSG_CUDA(cudaMalloc((void**)&sg->rowval, sizeof(float) * (n > 0 ? n : 1)));
    GSG_CUDA(cudaMalloc((void**)&sg->indptr, sizeof(int64_t) * (n + 1)));
    GSG_CUDA(cudaMalloc((void**)&sg->rowptr, sizeof(int32_t) * (n + 1)));
    GSG_CUDA(cudaMalloc((void**)&sg->perm, sizeof(int32_t) * (n > 0 ? n : 1)));
    sg->cap_n = n;
  }
  if (nnz > sg->cap_nnz) {
    cudaFree(sg->indices); cudaFree(sg->values);
    sg->indices = nullptr; sg->values = nullptr;
    GSG_CUDA(cudaMalloc((void**)&sg->indices, sizeof(int32_t) * nnz));
    sg->cap_nnz = nnz;
  }
  if (h_values && !sg->values) GSG_CUDA(cudaMalloc((void**)&sg->values, sizeof(float) * (sg->cap_nnz > 0 ? sg->cap_nnz : 1)));
  sg->n = n;
  sg->nnz = nnz;
  sg->norm_mode = -1;
  sg->dev_sized = false;
  sg->has_values = h_values != nullptr;
  // cudaMemcpyDefault: host (pinned or pageable) or device source arrays (UVA)
  GSG_CUDA(cudaMemcpyAsync(sg->indptr, h_indptr, sizeof(int64_t) * (n + 1), cudaMemcpyDefault, c->stream));
  if (nnz) GSG_CUDA(cudaMemcpyAsync(sg->indices, h_indices, sizeof(int32_t) * nnz, cudaMemcpyDefault, c->stream));
  if (h_values && nnz)
    GSG_CUDA(cudaMemcpyAsync(sg->values, h_values, sizeof(float) * nnz, cudaMemcpyDefault, c->stream));
  return GSG_OK;
}

GSG_API int gsg_gather_rows(gsg_ctx_t c, int32_t rows, int64_t row_bytes, const void* d_src, int64_t src_pitch,
                            const int32_t* d_idx, void* d_dst, int64_t dst_pitch) {
  if (int rc = check_ctx(c)) return rc;
  DeviceGuard dg(c->device);
  return gather_rows_launch(c, rows, row_bytes, d_src, src_pitch, d_idx, d_dst, dst_pitch);
}

GSG_API int gsg_subgraph_upload_device(gsg_ctx_t c, int32_t n, int64_t nnz, const int64_t* d_indptr,
                                       const int32_t* d_indices, const float* d_values, gsg_subgraph_t* out) {
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(out, GSG_EINVAL, "out is NULL");
  *out = nullptr;
  GSG_CHECK(d_indptr && (nnz == 0 || d_indices), GSG_EINVAL, "NULL indptr/indices");
  DeviceGuard dg(c->device);
  gsg_subgraph* sg = nullptr;
  if (int rc = alloc_subgraph(c, n, nnz, d_values != nullptr, &sg)) return rc;
  cudaError_t e = cudaMemcpyAsync(sg->indptr, d_indptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, c->stream);
  if (e == cudaSuccess && nnz)
    e = cudaMemcpyAsync(sg->indices, d_indices, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, c->stream);
  if (e == cudaSuccess && d_values && nnz)
    e = cudaMemcpyAsync(sg->values, d_values, sizeof(float) * nnz, cudaMemcpyDeviceToDevice, c->stream);
  if (e != cudaSuccess) { gsg_subgraph_free(sg); return cuda_fail(e, "cudaMemcpyAsync(upload_device)"); }
  *out = sg;
  return GSG_OK;
}

GSG_API int gsg_subgraph_create_device(gsg_ctx_t c, int32_t n, int64_t nnz_cap, gsg_subgraph_t* out) {
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(out, GSG_EINVAL, "out is NULL");
  *out = nullptr;
  GSG_CHECK(n >= 1 && nnz_cap >= 0, GSG_EINVAL, "bad device-sized subgraph n=%d nnz_cap=%lld", n, (long long)nnz_cap);
  DeviceGuard dg(c->device);
  gsg_subgraph* sg = nullptr;
  if (int rc = alloc_subgraph(c, n, nnz_cap, false, &sg)) return rc;
  sg->dev_sized = true;
  GSG_CUDA(cudaMemsetAsync(sg->indptr, 0, sizeof(int64_t) * (n + 1), c->stream));  // an empty graph until loaded
  *out = sg;
  return GSG_OK;
}

GSG_API int gsg_subgraph_normalize(gsg_ctx_t c, gsg_subgraph_t sg, int mode) {
  NvtxRange nvtx("gsg a1 normalize");
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(sg, GSG_EINVAL, "NULL subgraph");
  DeviceGuard dg(c->device);
  RowTag rt(c, GSG_K_A1);
  return normalize_launch(c, sg, mode);
}

GSG_API int gsg_subgraph_info(gsg_ctx_t c, gsg_subgraph_t sg, int32_t* n, int64_t* nnz_hat, int32_t* max_deg,
                              int32_t* n_heavy) {
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(sg, GSG_EINVAL, "NULL subgraph");
  DeviceGuard dg(c->device);
  GSG_CUDA(cudaStreamSynchronize(c->stream));
  int32_t cnt[2] = {0, 0};
  if (sg->norm_mode >= 0) GSG_CUDA(cudaMemcpy(cnt, sg->counters + kBins, sizeof(cnt), cudaMemcpyDeviceToHost));
  int32_t nh_dev = 0;  // device-sized subgraph: the entry count of Â is rowptr[n]
  if (sg->dev_sized && sg->norm_mode >= 0)
    GSG_CUDA(cudaMemcpy(&nh_dev, sg->rowptr + sg->n, sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (n) *n = sg->n;
  if (nnz_hat) *nnz_hat = sg->norm_mode >= 0 ? (sg->dev_sized ? (int64_t)nh_dev : sg->nnz_hat) : -1;
  if (max_deg) *max_deg = sg->norm_mode >= 0 ? cnt[1] : -1;
  if (n_heavy) *n_heavy = sg->norm_mode >= 0 ? cnt[0] : -1;
  return GSG_OK;
}

GSG_API int gsg_subgraph_download(gsg_ctx_t c, gsg_subgraph_t sg, int64_t* h_indptr, int32_t* h_idx, float* h_val,
                                  float* h_valT) {
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(sg && sg->norm_mode >= 0, GSG_EINVAL, "subgraph missing or not normalized");
  DeviceGuard dg(c->device);
  GSG_CUDA(cudaStreamSynchronize(c->stream));
  int64_t nh = sg->nnz_hat;
  if (sg->dev_sized) {
    int32_t v = 0;
    GSG_CUDA(cudaMemcpy(&v, sg->rowptr + sg->n, sizeof(int32_t), cudaMemcpyDeviceToHost));
    nh = v;
  }
  if (h_indptr) {
    std::vector<int32_t> tmp(sg->n + 1);
    GSG_CUDA(cudaMemcpy(tmp.data(), sg->rowptr, sizeof(int32_t) * (sg->n + 1), cudaMemcpyDeviceToHost));
    for (int32_t i = 0; i <= sg->n; i++) h_indptr[i] = tmp[i];
  }
  if (h_idx && nh) GSG_CUDA(cudaMemcpy(h_idx, sg->col, sizeof(int32_t) * nh, cudaMemcpyDeviceToHost));
  if (h_val && nh) GSG_CUDA(cudaMemcpy(h_val, sg->val, sizeof(float) * nh, cudaMemcpyDeviceToHost));
  if (h_valT && nh) GSG_CUDA(cudaMemcpy(h_valT, sg->valT, sizeof(float) * nh, cudaMemcpyDeviceToHost));
  int32_t err = 0;
  GSG_CUDA(cudaMemcpy(&err, sg->counters + 3 * kBins + 4, sizeof(int32_t), cudaMemcpyDeviceToHost));
  GSG_CHECK(err == 0, GSG_EGRAPH, "transpose values: a reverse edge was missing (asymmetric structure)");
  return GSG_OK;
}

GSG_API int gsg_subgraph_free(gsg_subgraph_t sg) {
  if (!sg) return GSG_OK;
  DeviceGuard dg(sg->device);
  cudaFree(sg->indptr); cudaFree(sg->indices); cudaFree(sg->values);
  cudaFree(sg->rowptr); cudaFree(sg->col); cudaFree(sg->val); cudaFree(sg->valT);
  cudaFree(sg->perm); cudaFree(sg->rowval); cudaFree(sg->counters); cudaFree(sg->rowid);
  cudaFree(sg->htask); cudaFree(sg->hcount);
  delete sg;
  return GSG_OK;
}

// ------------------------------------------------------------------------------ kernels
GSG_API int gsg_spmm(gsg_ctx_t c, gsg_subgraph_t sg, int transpose, int32_t f, const float* X, int64_t ldx, float* Y,
                     int64_t ldy, void* Ylp, int64_t ldylp, const float* mask, int64_t ldm, const uint32_t* mbits,
                     int64_t ldmb) {
  NvtxRange nvtx("gsg a2/a7 spmm");
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(sg, GSG_EINVAL, "NULL subgraph");
  DeviceGuard dg(c->device);
  BitsIO b;
  b.in = mbits;
  b.ldi = ldmb;
  return spmm_launch(c, sg, transpose ? 1 : 0, f, X, ldx, Y, ldy, Ylp, ldylp, mask, ldm, 0, 0, b);
}

GSG_API int gsg_gemm(gsg_ctx_t c, int32_t M, int32_t N, int32_t K, const void* A, int64_t lda, int transA, const void* B,
                     int64_t ldb, int transB, float* C, int64_t ldc, void* Clp, int64_t ldclp, int precision, int epilogue,
                     const float* aux, int64_t ldaux, const uint32_t* auxbits, int64_t ldauxb, uint32_t* Cbits,
                     int64_t ldcb, int split_k, int accumulate) {
  NvtxRange nvtx("gsg a3/a5/a6 gemm");
  if (int rc = check_ctx(c)) return rc;
  DeviceGuard dg(c->device);
  return gemm_launch(c, M, N, K, A, lda, transA ? 1 : 0, B, ldb, transB ? 1 : 0, C, ldc, Clp, ldclp, precision,
                     epilogue, aux, ldaux, split_k, accumulate, BitsIO{Cbits, ldcb, auxbits, ldauxb});
}

GSG_API int gsg_to_bf16(gsg_ctx_t c, int32_t rows, int32_t cols, const float* src, int64_t lds, void* dst, int64_t ldd) {
  if (int rc = check_ctx(c)) return rc;
  DeviceGuard dg(c->device);
  return to_bf16_launch(c, rows, cols, src, lds, dst, ldd);
}

GSG_API int gsg_layer_forward(gsg_ctx_t c, gsg_subgraph_t sg, int32_t f_in, int32_t f_out, const float* X, int64_t ldx,
                              const float* W, int64_t ldw, float* P, int64_t ldp, void* Plp, int64_t ldplp, float* H,
                              int64_t ldh, void* Hlp, int64_t ldhlp, uint32_t* Hbits, int64_t ldhbits, int precision,
                              int flags) {
  NvtxRange nvtx("gsg a2-a3 layer_forward");
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(sg, GSG_EINVAL, "NULL subgraph");
  GSG_CHECK(f_in >= 1 && f_out >= 1, GSG_EINVAL, "f_in=%d f_out=%d must be >= 1", f_in, f_out);
  GSG_CHECK(W && ldw >= f_out, GSG_EINVAL, "W NULL or ldw < f_out");
  GSG_CHECK(precision != GSG_PREC_BF16 || Plp || (flags & GSG_ORDER_A_XW), GSG_EINVAL,
            "BF16 forward needs the bf16 P copy (Plp)");
  GSG_CHECK(!Hbits || !(flags & GSG_NO_RELU), GSG_EINVAL, "the H bitmask needs the ReLU (not GSG_NO_RELU)");
  DeviceGuard dg(c->device);
  BitsIO hb;  // 1[H > 0] for the layer above's backward gate
  hb.out = Hbits;
  hb.ldo = ldhbits;
  const int n = sg->n;
  int rc;
  RowTag rt(c, GSG_K_A3);  // transform (a3); the aggregation calls below switch to a2
  if (flags & GSG_ORDER_A_XW) {
    // chain order 2 (§7.1): Y = X W (into P), H = ReLU(Â Y)
    GSG_CHECK(ldp >= f_out, GSG_EINVAL, "GSG_ORDER_A_XW: P holds Y = X W and needs ldp >= f_out");
    if (precision == GSG_PREC_BF16) {
      const int64_t ldxl = round_up(f_in, 8);
      const void* Wl = nullptr;
      int64_t ldwl2 = 0;
      if ((rc = bf16_weight(c, W, ldw, f_in, f_out, flags, &Wl, &ldwl2))) return rc;
      if ((rc = c->ws_lp2.reserve(sizeof(uint16_t) * n * ldxl))) return rc;
      if ((rc = to_bf16_launch(c, n, f_in, X, ldx, c->ws_lp2.ptr, ldxl))) return rc;
      rc = gemm_launch(c, n, f_out, f_in, c->ws_lp2.ptr, ldxl, 0, Wl, ldwl2, 0, P, ldp, nullptr, 0, precision,
                       GSG_EPI_NONE, nullptr, 0, 0, 0);
    } else {
      rc = gemm_launch(c, n, f_out, f_in, X, ldx, 0, W, ldw, 0, P, ldp, nullptr, 0, precision, GSG_EPI_NONE, nullptr, 0,
                       0, 0);
    }
    if (rc) return rc;
    c->prof_row = GSG_K_A2;
    return spmm_launch(c, sg, 0, f_out, P, ldp, H, ldh, Hlp, ldhlp, nullptr, 0, (flags & GSG_NO_RELU) ? 0 : 1, 0, hb);
  }
  c->prof_row = GSG_K_A2;
  rc = spmm_launch(c, sg, 0, f_in, X, ldx, P, ldp, precision == GSG_PREC_BF16 ? Plp : nullptr, ldplp, nullptr, 0);
  if (rc) return rc;
  c->prof_row = GSG_K_A3;
  const int epi = (flags & GSG_NO_RELU) ? GSG_EPI_NONE : GSG_EPI_RELU;
  if (precision == GSG_PREC_BF16) {
    const void* Wl = nullptr;
    int64_t ldwl = 0;
    if ((rc = bf16_weight(c, W, ldw, f_in, f_out, flags, &Wl, &ldwl))) return rc;
    return gemm_launch(c, n, f_out, f_in, Plp, ldplp, 0, Wl, ldwl, 0, H, ldh, Hlp, ldhlp, precision, epi,
                       nullptr, 0, 0, 0, hb);
  }
  return gemm_launch(c, n, f_out, f_in, P, ldp, 0, W, ldw, 0, H, ldh, Hlp, ldhlp, precision, epi, nullptr, 0, 0, 0, hb);
}

GSG_API int gsg_layer_backward(gsg_ctx_t c, gsg_subgraph_t sg, int32_t f_in, int32_t f_out, const float* P, int64_t ldp,
                               const void* Plp, int64_t ldplp, const float* H, int64_t ldh, const float* dH, int64_t lddh,
                               const void* dHlp, int64_t lddhlp, const float* W, int64_t ldw, float* dW, int64_t lddw,
                               float* dX, int64_t lddx, void* dXlp, int64_t lddxlp, const float* Hbelow, int64_t ldhb,
                               const uint32_t* Hbelow_bits, int64_t ldhbb, int precision, int flags) {
  NvtxRange nvtx("gsg a4-a7 layer_backward");
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(sg, GSG_EINVAL, "NULL subgraph");
  GSG_CHECK(f_in >= 1 && f_out >= 1, GSG_EINVAL, "f_in=%d f_out=%d must be >= 1", f_in, f_out);
  GSG_CHECK(P && dH && W && dW, GSG_EINVAL, "P, dH, W, dW must be non-NULL");
  GSG_CHECK((flags & GSG_DH_PREMASKED) || H, GSG_EINVAL, "H is needed unless GSG_DH_PREMASKED");
  GSG_CHECK(precision != GSG_PREC_BF16 || Plp, GSG_EINVAL, "BF16 backward needs the bf16 P copy (Plp)");
  GSG_CHECK(lddh >= f_out && lddh % 4 == 0, GSG_EINVAL, "lddh must be >= f_out and a multiple of 4");
  DeviceGuard dg(c->device);
  const int n = sg->n;
  const bool bf16 = precision == GSG_PREC_BF16;
  int rc;
  RowTag rt(c, GSG_K_A4);
  // the layer below's ReLU' gate: its bitmask (1/32 of the bytes) when given, else H_below itself
  BitsIO gb;
  gb.in = Hbelow_bits;
  gb.ldi = ldhbb;
  const bool gate = Hbelow || Hbelow_bits;
  // dZ = dH ⊙ 1[H > 0]   (row a4)
  const float* dZ = dH;
  int64_t lddz = lddh;
  const void* dZlp = dHlp;
  int64_t lddzlp = lddhlp;
  if (!(flags & GSG_DH_PREMASKED)) {
    // BF16 chain order 1 reads only the bf16 dZ (both GEMMs): the fp32 copy is not written
    const bool need_fp32 = !bf16 || (flags & GSG_ORDER_A_XW);
    lddz = round_up(f_out, 4);
    if (need_fp32 && (rc = c->ws_dZ.reserve(sizeof(float) * n * lddz))) return rc;
    void* lp = nullptr;
    if (bf16) {
      lddzlp = round_up(f_out, 8);
      if ((rc = c->ws_lp1.reserve(sizeof(uint16_t) * n * lddzlp))) return rc;
      lp = c->ws_lp1.ptr;
    }
    float* dzo = need_fp32 ? (float*)c->ws_dZ.ptr : nullptr;
    rc = (flags & GSG_H_BITS)
             ? mask_bits_launch(c, n, f_out, dH, lddh, reinterpret_cast<const uint32_t*>(H), ldh, dzo, lddz, lp, lddzlp)
             : mask_launch(c, n, f_out, dH, lddh, H, ldh, dzo, lddz, lp, lddzlp);
    if (rc) return rc;
    dZ = dzo;
    dZlp = lp;
  } else if (bf16 && !dZlp) {
    lddzlp = round_up(f_out, 8);
    if ((rc = c->ws_lp1.reserve(sizeof(uint16_t) * n * lddzlp))) return rc;
    if ((rc = to_bf16_launch(c, n, f_out, dH, lddh, c->ws_lp1.ptr, lddzlp))) return rc;
    dZlp = c->ws_lp1.ptr;
  }
  if (flags & GSG_ORDER_A_XW) {
    // chain order 2 backward: G = Âᵀ dZ (width f_out), dW = Xᵀ G, dX = (G Wᵀ) ⊙ 1[H_below > 0]; P holds X
    const int64_t ldg = round_up(f_out, 8);
    if ((rc = c->ws_T.reserve(sizeof(float) * n * ldg))) return rc;
    float* G = (float*)c->ws_T.ptr;
    void* Glp = nullptr;
    if (bf16) {
      if ((rc = c->ws_lp2.reserve(sizeof(uint16_t) * n * ldg))) return rc;
      Glp = c->ws_lp2.ptr;
    }
    c->prof_row = GSG_K_A7;
    if ((rc = spmm_launch(c, sg, 1, f_out, dZ, lddz, G, ldg, Glp, ldg, nullptr, 0))) return rc;
    c->prof_row = GSG_K_A5;
    const void* Wop2 = W;
    int64_t ldw2 = ldw;
    if (bf16 && (rc = bf16_weight(c, W, ldw, f_in, f_out, flags, &Wop2, &ldw2))) return rc;
    X3Lo glo_b, glo_a;  // FP32X3: G's lo once for dW (B = G) and dX (A = G)
    if (precision == GSG_PREC_FP32X3 && x3_implicit() && n > 0) {
      const int64_t ldl = round_up(f_out, 4);
      if ((rc = c->ws_x3dz.reserve(sizeof(float) * n * ldl))) return rc;
      if ((rc = split_lo_launch(c, n, f_out, G, ldg, (float*)c->ws_x3dz.ptr, ldl))) return rc;
      glo_b.b = glo_a.a = (const float*)c->ws_x3dz.ptr;
      glo_b.ldb = glo_a.lda = ldl;
    }
    rc = gemm_launch(c, f_in, f_out, n, bf16 ? Plp : (const void*)P, bf16 ? ldplp : ldp, 1, bf16 ? Glp : (const void*)G,
                     ldg, 0, dW, lddw, nullptr, 0, precision, GSG_EPI_NONE, nullptr, 0, 0, (flags & GSG_ACCUM_DW) ? 1 : 0,
                     BitsIO{}, glo_b);
    if (rc || !dX) return rc;
    c->prof_row = GSG_K_A6;
    return gemm_launch(c, n, f_in, f_out, bf16 ? Glp : (const void*)G, ldg, 0, Wop2, ldw2, 1, dX, lddx, dXlp, lddxlp,
                       precision, gate ? GSG_EPI_MASK : GSG_EPI_NONE, Hbelow, ldhb, 0, 0, gb, glo_a);
  }
  const void* Wop = W;
  int64_t ldwop = ldw;
  c->prof_row = GSG_K_A6;
  if (bf16 && (rc = bf16_weight(c, W, ldw, f_in, f_out, flags, &Wop, &ldwop))) return rc;
  c->prof_row = GSG_K_A5;
  // dW = Pᵀ dZ (row a5) and T = dZ Wᵀ -> dX (rows a6, a7) only share read-only inputs: the dW
  // GEMM runs on the context's side stream (fork / join by events, also inside a CUDA-graph
  // capture), overlapping its fill / drain and split-K reduction with T's GEMM (config 5: -15 us
  // per step, configs 3-4 -0.2-0.7 %, config 2 +1 %). GSG_BWD_FORK=0 serializes them (A/B);
  // profiling serializes too (clean per-stage events).
  // FP32X3: dZ's lo is split once for both GEMMs (it is B of dW and A of T, the same stored matrix)
  X3Lo dzlo;
  if (precision == GSG_PREC_FP32X3 && x3_implicit() && n > 0 && f_out > 0) {
    const int64_t ldl = round_up(f_out, 4);
    if ((rc = c->ws_x3dz.reserve(sizeof(float) * n * ldl))) return rc;
    if ((rc = split_lo_launch(c, n, f_out, dZ, lddz, (float*)c->ws_x3dz.ptr, ldl))) return rc;
    dzlo.a = dzlo.b = (const float*)c->ws_x3dz.ptr;
    dzlo.lda = dzlo.ldb = ldl;
  }
  SideFork fk(c, fork_enabled() && dX && !c->prof.on);
  const int64_t ldt = round_up(f_in, 4);
  float* T = nullptr;
  X3Lo dzlo_a;
  dzlo_a.a = dzlo.a;
  dzlo_a.lda = dzlo.lda;
  // T = dZ Wᵀ   (row a6): A = dZ (K-major), B = W stored f_in x f_out = N x K (K-major)
  auto launch_T = [&]() -> int {
    c->prof_row = GSG_K_A6;
    if (int r = c->ws_T.reserve(sizeof(float) * n * ldt)) return r;
    T = (float*)c->ws_T.ptr;
    return gemm_launch(c, n, f_in, f_out, bf16 ? dZlp : (const void*)dZ, bf16 ? lddzlp : lddz, 0, Wop, ldwop, 1, T,
                       ldt, nullptr, 0, precision, GSG_EPI_NONE, nullptr, 0, 0, 0, BitsIO{}, dzlo_a);
  };
  // GSG_BWD_TFIRST (A/B): T is enqueued on the main stream before the forked dW (both wait only
  // for dZ), so T's CTAs take the SMs first and dW fills them as T's tiles run out
  const bool tfirst = fk.away && t_first(f_in, f_out);
  if (tfirst) {
    c->stream = fk.main;
    rc = launch_T();
    c->stream = c->side;
    if (rc) return rc;
  }
  c->prof_row = GSG_K_A5;
  // dW = Pᵀ dZ   (row a5): A = P stored n x f_in (MN-major), B = dZ stored n x f_out (MN-major)
  c->side_ws = true;
  X3Lo dzlo_b;
  dzlo_b.b = dzlo.b;
  dzlo_b.ldb = dzlo.ldb;
  rc = gemm_launch(c, f_in, f_out, n, bf16 ? Plp : (const void*)P, bf16 ? ldplp : ldp, 1, bf16 ? dZlp : (const void*)dZ,
                   bf16 ? lddzlp : lddz, 0, dW, lddw, nullptr, 0, precision, GSG_EPI_NONE, nullptr, 0, 0,
                   (flags & GSG_ACCUM_DW) ? 1 : 0, BitsIO{}, dzlo_b);
  c->side_ws = false;
  fk.back();
  if (rc) return rc;
  if (!dX) return GSG_OK;
  if (!tfirst && (rc = launch_T())) return rc;
  // dX = Âᵀ T [⊙ 1[H_below > 0]]   (row a7, fused a4 of the layer below)
  c->prof_row = GSG_K_A7;
  return spmm_launch(c, sg, 1, f_in, T, ldt, dX, lddx, dXlp, lddxlp, Hbelow, ldhb, 0, 0, gb);  // fk joins on exit
}

GSG_API int gsg_sage_forward(gsg_ctx_t c, gsg_subgraph_t sg, int32_t f_in, int32_t fh, const float* X, int64_t ldx,
                             const float* Ws, int64_t ldws, const float* Wn, int64_t ldwn, float* P, int64_t ldp,
                             float* H, int64_t ldh, int precision, int flags) {
  NvtxRange nvtx("gsg sage_forward");
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(sg, GSG_EINVAL, "NULL subgraph");
  GSG_CHECK(precision == GSG_PREC_TF32 || precision == GSG_PREC_FP32X3, GSG_EUNSUPPORTED,
            "GraphSAGE layer: TF32 or FP32X3 only");
  GSG_CHECK(f_in >= 1 && fh >= 1 && fh % 4 == 0, GSG_EINVAL, "f_in=%d f_half=%d (f_half %% 4 == 0 required)", f_in, fh);
  GSG_CHECK(X && Ws && Wn && P && H && ldh >= 2 * fh, GSG_EINVAL, "NULL argument or ldh < 2 f_half");
  DeviceGuard dg(c->device);
  const int n = sg->n;
  const int epi = (flags & GSG_NO_RELU) ? GSG_EPI_NONE : GSG_EPI_RELU;
  int rc = spmm_launch(c, sg, 0, f_in, X, ldx, P, ldp, nullptr, 0, nullptr, 0);  // P = Ã X
  if (rc) return rc;
  rc = gemm_launch(c, n, fh, f_in, X, ldx, 0, Ws, ldws, 0, H, ldh, nullptr, 0, precision, epi, nullptr, 0, 0, 0);
  if (rc) return rc;
  return gemm_launch(c, n, fh, f_in, P, ldp, 0, Wn, ldwn, 0, H + fh, ldh, nullptr, 0, precision, epi, nullptr, 0, 0, 0);
}

GSG_API int gsg_sage_backward(gsg_ctx_t c, gsg_subgraph_t sg, int32_t f_in, int32_t fh, const float* X, int64_t ldx,
                              const float* P, int64_t ldp, const float* H, int64_t ldh, const float* dH, int64_t lddh,
                              const float* Ws, int64_t ldws, const float* Wn, int64_t ldwn, float* dWs, int64_t lddws,
                              float* dWn, int64_t lddwn, float* dX, int64_t lddx, const float* Hbelow, int64_t ldhb,
                              int precision, int flags) {
  NvtxRange nvtx("gsg sage_backward");
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(sg, GSG_EINVAL, "NULL subgraph");
  GSG_CHECK(precision == GSG_PREC_TF32 || precision == GSG_PREC_FP32X3, GSG_EUNSUPPORTED,
            "GraphSAGE layer: TF32 or FP32X3 only");
  GSG_CHECK(f_in >= 1 && fh >= 1 && fh % 4 == 0, GSG_EINVAL, "f_in=%d f_half=%d (f_half %% 4 == 0 required)", f_in, fh);
  GSG_CHECK(X && P && dH && Ws && Wn && dWs && dWn, GSG_EINVAL, "NULL argument");
  GSG_CHECK((flags & GSG_DH_PREMASKED) || H, GSG_EINVAL, "H is needed unless GSG_DH_PREMASKED");
  GSG_CHECK(!(flags & GSG_H_BITS), GSG_EUNSUPPORTED, "GSG_H_BITS is a gsg_layer_backward flag");
  GSG_CHECK(lddh >= 2 * fh && lddh % 4 == 0, GSG_EINVAL, "lddh must be >= 2 f_half and a multiple of 4");
  DeviceGuard dg(c->device);
  const int n = sg->n;
  int rc;
  const float* dZ = dH;
  int64_t lddz = lddh;
  if (!(flags & GSG_DH_PREMASKED)) {
    lddz = round_up(2 * fh, 4);
    if ((rc = c->ws_dZ.reserve(sizeof(float) * n * lddz))) return rc;
    if ((rc = mask_launch(c, n, 2 * fh, dH, lddh, H, ldh, (float*)c->ws_dZ.ptr, lddz, nullptr, 0))) return rc;
    dZ = (const float*)c->ws_dZ.ptr;
  }
  const float* dZs = dZ;        // self half    (Eq. 12 / 14 slice [:, 0:f/2])
  const float* dZn = dZ + fh;   // neighbor half (Eq. 13 / 15 slice [:, f/2:f])
  // dW_s = Xᵀ dZ_s ; dW_n = Pᵀ dZ_n   (Eqs. 12-13)
  rc = gemm_launch(c, f_in, fh, n, X, ldx, 1, dZs, lddz, 0, dWs, lddws, nullptr, 0, precision, GSG_EPI_NONE, nullptr, 0,
                   0, (flags & GSG_ACCUM_DW) ? 1 : 0);
  if (rc) return rc;
  rc = gemm_launch(c, f_in, fh, n, P, ldp, 1, dZn, lddz, 0, dWn, lddwn, nullptr, 0, precision, GSG_EPI_NONE, nullptr, 0,
                   0, (flags & GSG_ACCUM_DW) ? 1 : 0);
  if (rc || !dX) return rc;
  // dX = dZ_s W_sᵀ + Ãᵀ (dZ_n W_nᵀ), gated by H_below   (Eqs. 14-15)
  const int64_t ldt = round_up(f_in, 4);
  if ((rc = c->ws_T.reserve(sizeof(float) * n * ldt))) return rc;
  float* T = (float*)c->ws_T.ptr;
  rc = gemm_launch(c, n, f_in, fh, dZn, lddz, 0, Wn, ldwn, 1, T, ldt, nullptr, 0, precision, GSG_EPI_NONE, nullptr, 0, 0,
                   0);
  if (rc) return rc;
  rc = gemm_launch(c, n, f_in, fh, dZs, lddz, 0, Ws, ldws, 1, dX, lddx, nullptr, 0, precision, GSG_EPI_NONE, nullptr, 0,
                   0, 0);
  if (rc) return rc;
  return spmm_launch(c, sg, 1, f_in, T, ldt, dX, lddx, nullptr, 0, Hbelow, ldhb, 0, /*accum=*/1);
}

GSG_API int gsg_head(gsg_ctx_t c, int32_t n, int32_t f, int32_t C, int kind, const float* HL, int64_t ldh,
                     const float* Wm, int64_t ldw, const void* labels, float* S, float* dS, int64_t lds, float* dWm,
                     int64_t lddw, float* dHL, int64_t lddh, void* dHlp, int64_t lddhlp, float* loss, int precision,
                     const float* node_w, const uint32_t* HLbits, int64_t ldhlb) {
  NvtxRange nvtx("gsg a8 head");
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(kind == GSG_HEAD_SOFTMAX || kind == GSG_HEAD_SIGMOID, GSG_EINVAL, "bad head kind %d", kind);
  GSG_CHECK(n >= 1 && f >= 1 && C >= 1, GSG_EINVAL, "bad head sizes n=%d f=%d C=%d", n, f, C);
  GSG_CHECK(HL && Wm && labels && S && dS && dWm && dHL && loss, GSG_EINVAL, "NULL head argument");
  GSG_CHECK(lds >= C && lds % 4 == 0, GSG_EINVAL, "lds must be >= C and a multiple of 4");
  // the head runs in TF32 (H_L is fp32, C is small; SUPPORT), or 3xTF32 when asked
  const int hp = precision == GSG_PREC_FP32X3 ? GSG_PREC_FP32X3 : GSG_PREC_TF32;
  DeviceGuard dg(c->device);
  RowTag rt(c, GSG_K_A8);
  // FP32X3: H_L's lo serves S (A = H_L) and dW_mlp (A = H_Lᵀ, the same stored matrix), dS's lo
  // dW_mlp (B) and dH_L (A): each split once
  const bool x3pre = hp == GSG_PREC_FP32X3 && x3_implicit() && n > 0;
  X3Lo hl_lo, ds_lo;
  int rc;
  if (x3pre) {
    const int64_t ldl = round_up(f, 4);
    if ((rc = c->ws_x3hl.reserve(sizeof(float) * n * ldl))) return rc;
    if ((rc = split_lo_launch(c, n, f, HL, ldh, (float*)c->ws_x3hl.ptr, ldl))) return rc;
    hl_lo.a = (const float*)c->ws_x3hl.ptr;
    hl_lo.lda = ldl;
  }
  rc = gemm_launch(c, n, C, f, HL, ldh, 0, Wm, ldw, 0, S, lds, nullptr, 0, hp, GSG_EPI_NONE, nullptr, 0, 0, 0,
                   BitsIO{}, hl_lo);
  if (rc) return rc;
  if ((rc = head_loss_launch(c, n, C, kind, S, lds, labels, node_w, dS, loss))) return rc;
  if (x3pre) {
    const int64_t ldl = round_up(C, 4);
    if ((rc = c->ws_x3dz.reserve(sizeof(float) * n * ldl))) return rc;
    if ((rc = split_lo_launch(c, n, C, dS, lds, (float*)c->ws_x3dz.ptr, ldl))) return rc;
    ds_lo.a = ds_lo.b = (const float*)c->ws_x3dz.ptr;
    ds_lo.lda = ds_lo.ldb = ldl;
  }
  X3Lo dwm_lo = hl_lo;  // dW_mlp = H_Lᵀ dS: A = H_L, B = dS
  dwm_lo.b = ds_lo.b;
  dwm_lo.ldb = ds_lo.ldb;
  X3Lo dhl_lo;  // dH_L = dS W_mlpᵀ: A = dS
  dhl_lo.a = ds_lo.a;
  dhl_lo.lda = ds_lo.lda;
  // dW_mlp = H_Lᵀ dS and dH_L = (dS W_mlpᵀ) ⊙ 1[H_L > 0] only share read-only inputs: the first
  // runs on the side stream (fork / join, as in gsg_layer_backward; serialized while profiling)
  SideFork fk(c, fork_enabled() && !c->prof.on);
  BitsIO gb;  // ReLU' gate of H_L: its bitmask when given
  gb.in = HLbits;
  gb.ldi = ldhlb;
  auto launch_dHL = [&]() {
    return gemm_launch(c, n, f, C, dS, lds, 0, Wm, ldw, 1, dHL, lddh, dHlp, lddhlp, hp, GSG_EPI_MASK, HL, ldh, 0, 0,
                       gb, dhl_lo);
  };
  const bool dh_first = fk.away && head_dh_first();
  if (dh_first) {  // GSG_HEAD_DHFIRST (A/B): dH_L enqueued on the main stream before the forked dW_mlp
    c->stream = fk.main;
    rc = launch_dHL();
    c->stream = c->side;
    if (rc) return rc;
  }
  c->side_ws = true;
  rc = gemm_launch(c, f, C, n, HL, ldh, 1, dS, lds, 0, dWm, lddw, nullptr, 0, hp, GSG_EPI_NONE, nullptr, 0, 0, 0,
                   BitsIO{}, dwm_lo);
  c->side_ws = false;
  fk.back();
  if (rc) return rc;
  return dh_first ? GSG_OK : launch_dHL();  // fk joins on exit
}

// ------------------------------------------------------------------------------ NCCL
GSG_API int gsg_nccl_unique_id(void* out) {
  GSG_CHECK(out, GSG_EINVAL, "out is NULL");
  Nccl& N = nccl();
  GSG_CHECK(N.ok, GSG_ENCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  ncclResult_t r = N.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
  return GSG_OK;
}

GSG_API int gsg_nccl_comm_init(gsg_ctx_t c, int nranks, int rank, const void* id128, void** out) {
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(out && id128 && nranks >= 1 && rank >= 0 && rank < nranks, GSG_EINVAL, "bad comm_init arguments");
  Nccl& N = nccl();
  GSG_CHECK(N.ok, GSG_ENCCL, "libnccl.so.2 not loadable");
  DeviceGuard dg(c->device);
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t comm;
  ncclResult_t r = N.CommInitRank(&comm, nranks, id, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *out = comm;
  return GSG_OK;
}

GSG_API int gsg_nccl_comm_destroy(void* comm) {
  if (!comm) return GSG_OK;
  Nccl& N = nccl();
  GSG_CHECK(N.ok, GSG_ENCCL, "libnccl.so.2 not loadable");
  ncclResult_t r = N.CommDestroy(static_cast<ncclComm_t>(comm));
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return GSG_OK;
}

GSG_API int gsg_allreduce_grads(gsg_ctx_t c, void* comm, float* const* bufs, const int64_t* counts, int nbufs,
                                int average) {
  NvtxRange nvtx("gsg a9 allreduce_grads");
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(comm && bufs && counts && nbufs >= 0, GSG_EINVAL, "bad allreduce arguments");
  Nccl& N = nccl();
  GSG_CHECK(N.ok, GSG_ENCCL, "libnccl.so.2 not loadable");
  DeviceGuard dg(c->device);
  ncclResult_t ae = ncclSuccess;  // an earlier collective failed asynchronously: report it, enqueue nothing
  if (N.CommGetAsyncError(static_cast<ncclComm_t>(comm), &ae) == ncclSuccess && ae != ncclSuccess &&
      ae != ncclInProgress)
    return nccl_fail(ae, "NCCL communicator in an asynchronous error state (earlier collective)");
  ncclResult_t r = N.GroupStart();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
  for (int i = 0; i < nbufs; i++) {
    if (counts[i] <= 0) continue;
    r = N.AllReduce(bufs[i], bufs[i], (size_t)counts[i], ncclFloat32, average ? ncclAvg : ncclSum,
                    static_cast<ncclComm_t>(comm), c->stream);
    if (r != ncclSuccess) { N.GroupEnd(); return nccl_fail(r, "ncclAllReduce"); }
  }
  r = N.GroupEnd();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
  return GSG_OK;
}

GSG_API int gsg_nccl_wait(gsg_ctx_t c, void* comm, int64_t timeout_ms) {
  NvtxRange nvtx("gsg a9 nccl_wait");
  if (int rc = check_ctx(c)) return rc;
  GSG_CHECK(comm, GSG_EINVAL, "NULL communicator");
  Nccl& N = nccl();
  GSG_CHECK(N.ok, GSG_ENCCL, "libnccl.so.2 not loadable");
  DeviceGuard dg(c->device);
  ncclComm_t cm = static_cast<ncclComm_t>(comm);
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(c->stream);
    ncclResult_t ae = ncclSuccess;
    const ncclResult_t qr = N.CommGetAsyncError(cm, &ae);
    if (qr != ncclSuccess) return nccl_fail(qr, "ncclCommGetAsyncError");
    if (ae != ncclSuccess && ae != ncclInProgress) {
      N.CommAbort(cm);
      return nccl_fail(ae, "NCCL asynchronous error (communicator aborted)");
    }
    if (q == cudaSuccess) return GSG_OK;
    if (q != cudaErrorNotReady) return cuda_fail(q, "cudaStreamQuery(gsg_nccl_wait)");
    const int64_t ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_ms > 0 && ms > timeout_ms) {
      N.CommAbort(cm);
      return fail(GSG_ENCCL, "gsg_nccl_wait: stream not done after %lld ms (a peer rank stalled or died?); "
                             "communicator aborted", (long long)ms);
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

}  // extern "C"
