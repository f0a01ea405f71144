"""Thin Python binding of libgsg.so (include/gsg.h): the B200-native GCN-layer hot path of
graph-sampling GNN training (arXiv 2010.03166).

Argument marshalling only: every compute step runs in the library's sm_100a kernels. The
``gsg_*`` functions mirror the C ABI one-to-one (integers for pointers); ``Context`` and
``Subgraph`` add torch-tensor conveniences (``tensor.data_ptr()``, row strides) on top.
There is no CPU fallback: importing this package fails loudly if libgsg.so is missing, and
creating a context fails on anything but a CUDA device of compute capability 10.0.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GSG_LIB_PATH: load another build of the same library (A/B measurements of two builds in one run)
LIB_PATH = os.environ.get("GSG_LIB_PATH") or os.path.join(_HERE, "libgsg.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "gsg.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make gsg` (or __graft_entry__.build()); "
                      "there is no fallback implementation")

_lib = ctypes.CDLL(LIB_PATH)

# ---- constants (gsg.h) ----
GSG_OK, GSG_EINVAL, GSG_EGRAPH, GSG_ENOMEM, GSG_ECUDA, GSG_ENCCL, GSG_EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
GSG_NORM_ROW_SELF, GSG_NORM_SYM_SELF, GSG_NORM_ROW, GSG_NORM_VALUES = 0, 1, 2, 3
GSG_PREC_TF32, GSG_PREC_BF16, GSG_PREC_FP32X3 = 0, 1, 2
GSG_NO_RELU, GSG_DH_PREMASKED, GSG_ACCUM_DW, GSG_ORDER_A_XW, GSG_W_BF16, GSG_H_BITS = 1, 2, 4, 8, 16, 32
GSG_EPI_NONE, GSG_EPI_RELU, GSG_EPI_MASK = 0, 1, 2
GSG_HEAD_SOFTMAX, GSG_HEAD_SIGMOID = 0, 1
GSG_K_SPMM, GSG_K_GEMM, GSG_K_NORM, GSG_K_OTHER = 0, 1, 2, 3
# the same launches by SURVEY §8(a) row (gsg.h): a1 normalize ... a8 head
GSG_K_A1, GSG_K_A2, GSG_K_A3, GSG_K_A4, GSG_K_A5, GSG_K_A6, GSG_K_A7, GSG_K_A8 = range(4, 12)
GSG_K_CLASSES = 12

_vp, _i32, _i64, _int = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int
_SIGS = {
    "gsg_ctx_create": (_int, [_int, _vp, ctypes.POINTER(_vp)]),
    "gsg_ctx_destroy": (_int, [_vp]),
    "gsg_ctx_set_stream": (_int, [_vp, _vp]),
    "gsg_ctx_stream": (_vp, [_vp]),
    "gsg_ctx_sync": (_int, [_vp]),
    "gsg_ctx_launch_count": (_i64, [_vp]),
    "gsg_last_error": (ctypes.c_char_p, []),
    "gsg_ctx_profile": (_int, [_vp, _int]),
    "gsg_ctx_profile_read": (_int, [_vp, _int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64),
                                    ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "gsg_subgraph_assign": (_int, [_vp, _vp, _i32, _i64, _vp, _vp, _vp, _int]),
    "gsg_subgraph_upload": (_int, [_vp, _i32, _i64, _vp, _vp, _vp, _int, ctypes.POINTER(_vp)]),
    "gsg_subgraph_upload_device": (_int, [_vp, _i32, _i64, _vp, _vp, _vp, ctypes.POINTER(_vp)]),
    "gsg_subgraph_normalize": (_int, [_vp, _vp, _int]),
    "gsg_subgraph_info": (_int, [_vp, _vp, ctypes.POINTER(_i32), ctypes.POINTER(_i64), ctypes.POINTER(_i32),
                                 ctypes.POINTER(_i32)]),
    "gsg_subgraph_download": (_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "gsg_subgraph_free": (_int, [_vp]),
    "gsg_spmm": (_int, [_vp, _vp, _int, _i32, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64]),
    "gsg_gemm": (_int, [_vp, _i32, _i32, _i32, _vp, _i64, _int, _vp, _i64, _int, _vp, _i64, _vp, _i64, _int, _int,
                        _vp, _i64, _vp, _i64, _vp, _i64, _int, _int]),
    "gsg_to_bf16": (_int, [_vp, _i32, _i32, _vp, _i64, _vp, _i64]),
    "gsg_layer_forward": (_int, [_vp, _vp, _i32, _i32, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp,
                                 _i64, _vp, _i64, _int, _int]),
    "gsg_layer_backward": (_int, [_vp, _vp, _i32, _i32, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp,
                                  _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _int, _int]),
    "gsg_head": (_int, [_vp, _i32, _i32, _i32, _int, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _i64, _vp, _i64, _vp, _i64,
                        _vp, _i64, _vp, _int, _vp, _vp, _i64]),
    "gsg_sage_forward": (_int, [_vp, _vp, _i32, _i32, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _int,
                                _int]),
    "gsg_sage_backward": (_int, [_vp, _vp, _i32, _i32, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp,
                                 _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _int, _int]),
    "gsg_parent_upload": (_int, [_vp, _i64, _i64, _vp, _vp, ctypes.POINTER(_vp)]),
    "gsg_parent_free": (_int, [_vp]),
    "gsg_frontier_sample": (_int, [_vp, _vp, _i32, _i32, _i32, ctypes.c_uint64, _i32, ctypes.POINTER(_vp)]),
    "gsg_gather_rows": (_int, [_vp, _i32, _i64, _vp, _i64, _vp, _vp, _i64]),
    "gsg_ctx_wait_event": (_int, [_vp, _vp]),
    "gsg_sample_get": (_int, [_vp, _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i64), ctypes.POINTER(_vp),
                              ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    "gsg_sample_free": (_int, [_vp]),
    "gsg_nccl_unique_id": (_int, [_vp]),
    "gsg_nccl_comm_init": (_int, [_vp, _int, _int, _vp, ctypes.POINTER(_vp)]),
    "gsg_nccl_comm_destroy": (_int, [_vp]),
    "gsg_allreduce_grads": (_int, [_vp, _vp, _vp, _vp, _int, _int]),
    "gsg_nccl_wait": (_int, [_vp, _vp, _i64]),
    "gsg_subgraph_create_device": (_int, [_vp, _i32, _i64, ctypes.POINTER(_vp)]),
    "gsg_sample_load": (_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "gsg_sample_check": (_int, [_vp]),
    "gsg_diag_gather_ceiling": (_int, [_vp, _vp, _i32, _i64, _i32, ctypes.POINTER(ctypes.c_double)]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f


class GsgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"gsg error {code}: {msg}")
        self.code = code


def last_error() -> str:
    return (gsg_last_error() or b"").decode(errors="replace")


def check(rc: int):
    if rc != GSG_OK:
        raise GsgError(rc, last_error())
    return rc


def exported_symbols():
    """Names declared with GSG_API in include/gsg.h (used by the not-gpu symbol test)."""
    import re
    txt = open(HEADER_PATH).read()
    return re.findall(r"GSG_API\s+[\w\s\*]+?\b(gsg_\w+)\s*\(", txt)


# ------------------------------------------------------------------------------ helpers
def _ptr(t) -> int:
    if t is None:
        return 0
    return int(t.data_ptr())


def _ld(t) -> int:
    if t is None:
        return 0
    assert t.dim() == 2 and t.stride(1) == 1, "row-major 2-D tensor with unit column stride expected"
    return int(t.stride(0))


class Subgraph:
    """Owning handle of a device subgraph (gsg_subgraph_t)."""

    def __init__(self, ctx: "Context", handle: int, n: int, nnz: int):
        self.ctx, self.h, self.n, self.nnz = ctx, handle, n, nnz

    def normalize(self, mode: int = GSG_NORM_ROW_SELF):
        check(gsg_subgraph_normalize(self.ctx.h, self.h, mode))
        return self

    def info(self):
        n, nh, md, nhv = _i32(), _i64(), _i32(), _i32()
        check(gsg_subgraph_info(self.ctx.h, self.h, ctypes.byref(n), ctypes.byref(nh), ctypes.byref(md),
                                ctypes.byref(nhv)))
        return {"n": n.value, "nnz_hat": nh.value, "max_deg_hat": md.value, "n_heavy": nhv.value}

    def download(self):
        inf = self.info()
        nh = inf["nnz_hat"]
        ip = np.empty(self.n + 1, np.int64)
        ix = np.empty(max(nh, 1), np.int32)
        v = np.empty(max(nh, 1), np.float32)
        vt = np.empty(max(nh, 1), np.float32)
        check(gsg_subgraph_download(self.ctx.h, self.h, ip.ctypes.data, ix.ctypes.data, v.ctypes.data, vt.ctypes.data))
        return ip, ix[:nh], v[:nh], vt[:nh]

    def assign(self, n: int, nnz: int, indptr_ptr: int, indices_ptr: int, values_ptr: int = 0, validate=False,
               ctx: "Context | None" = None):
        """Refill from host arrays given as raw pointers (pinned memory -> async copies), on the
        stream of `ctx` (default: the owning context), e.g. a copy stream overlapping compute."""
        c = self.ctx if ctx is None else ctx
        check(gsg_subgraph_assign(c.h, self.h, n, nnz, indptr_ptr, indices_ptr or None, values_ptr or None,
                                  int(validate)))
        self.n, self.nnz = n, nnz
        return self

    def free(self):
        if self.h:
            gsg_subgraph_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class ParentGraph:
    """Device-resident parent graph for GPU frontier sampling (gsg_parent_t)."""

    def __init__(self, ctx: "Context", indptr: np.ndarray, indices: np.ndarray):
        ip = np.ascontiguousarray(indptr, dtype=np.int64)
        ix = np.ascontiguousarray(indices, dtype=np.int32)
        h = _vp()
        check(gsg_parent_upload(ctx.h, ip.shape[0] - 1, int(ip[-1]), ip.ctypes.data, ix.ctypes.data, ctypes.byref(h)))
        self.ctx, self.h = ctx, h.value

    def sample(self, n: int, m: int, seed: int, count: int = 1, clip: int = 16) -> "SampleBatch":
        out = _vp()
        check(gsg_frontier_sample(self.ctx.h, self.h, n, m, clip, seed, count, ctypes.byref(out)))
        return SampleBatch(out.value, count)

    def free(self):
        if self.h:
            gsg_parent_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class SampleBatch:
    """`count` GPU-sampled, induced subgraphs (gsg_sample_t)."""

    def __init__(self, handle: int, count: int):
        self.h, self.count = handle, count

    def get(self, k: int) -> dict:
        n, nnz, ip, ix, nd = _i32(), _i64(), _vp(), _vp(), _vp()
        check(gsg_sample_get(self.h, k, ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(ip), ctypes.byref(ix),
                             ctypes.byref(nd)))
        return {"n": n.value, "nnz": nnz.value, "d_indptr": ip.value or 0, "d_indices": ix.value or 0,
                "d_nodes": nd.value or 0}

    def tensors(self, k: int):
        """Zero-copy torch views of sample k: (indptr int64 [n+1], indices int32 [nnz], nodes int32 [n])."""
        import torch
        v = self.get(k)
        n, nnz = v["n"], v["nnz"]
        return (torch.as_tensor(_DevView(v["d_indptr"], n + 1, "<i8"), device="cuda"),
                torch.as_tensor(_DevView(v["d_indices"], nnz, "<i4"), device="cuda"),
                torch.as_tensor(_DevView(v["d_nodes"], n, "<i4"), device="cuda"))

    def to_host(self, k: int):
        """Copy sample k back (tests): (indptr int64, indices int32, nodes int32) numpy arrays."""
        return tuple(t.cpu().numpy() for t in self.tensors(k))

    def load(self, ctx: "Context", d_k, sg: "Subgraph", nodes_out=None, node_w=None):
        """gsg_sample_load: sample d_k[0] (device int32 tensor) into the device-sized subgraph sg,
        then d_k[0] = (d_k[0] + 1) % count. Graph-capturable."""
        check(gsg_sample_load(ctx.h, self.h, _ptr(d_k), sg.h, _ptr(nodes_out) or None, _ptr(node_w) or None))

    def check(self):
        check(gsg_sample_check(self.h))

    def free(self):
        if self.h:
            gsg_sample_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class _DevView:
    """__cuda_array_interface__ wrapper of a library-owned device array (no copy)."""

    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (ptr or 0, False),
                                         "version": 3, "strides": None}


class Context:
    """gsg_ctx_t on one device; launches go to `stream` (a torch.cuda.Stream or raw handle)."""

    def __init__(self, device: int = 0, stream=None):
        """stream: torch.cuda.Stream or raw cudaStream_t; None = torch's current stream."""
        h = _vp()
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(device) if torch.cuda.is_available() else 0
        raw = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        check(gsg_ctx_create(device, raw or None, ctypes.byref(h)))
        self.h = h.value
        self.device = device

    @property
    def stream(self) -> int:
        return gsg_ctx_stream(self.h) or 0

    def set_stream(self, stream):
        raw = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        check(gsg_ctx_set_stream(self.h, raw))

    def sync(self):
        check(gsg_ctx_sync(self.h))

    def launch_count(self) -> int:
        return int(gsg_ctx_launch_count(self.h))

    def profile(self, enable: bool = True):
        check(gsg_ctx_profile(self.h, int(enable)))

    def profile_read(self, kclass: int) -> dict:
        ms, n, b, f = ctypes.c_double(), _i64(), ctypes.c_double(), ctypes.c_double()
        check(gsg_ctx_profile_read(self.h, kclass, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(b), ctypes.byref(f)))
        return {"ms": ms.value, "launches": n.value, "alg_bytes": b.value, "alg_flops": f.value}

    def close(self):
        if getattr(self, "h", None):
            gsg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- subgraph ----
    def upload(self, indptr: np.ndarray, indices: np.ndarray, values=None, validate: bool = True) -> Subgraph:
        ip = np.ascontiguousarray(indptr, dtype=np.int64)
        ix = np.ascontiguousarray(indices, dtype=np.int32)
        vals = None if values is None else np.ascontiguousarray(values, dtype=np.float32)
        n = ip.shape[0] - 1
        out = _vp()
        check(gsg_subgraph_upload(self.h, n, int(ip[-1]), ip.ctypes.data, ix.ctypes.data if ix.size else None,
                                  vals.ctypes.data if vals is not None else None, int(validate), ctypes.byref(out)))
        return Subgraph(self, out.value, n, int(ip[-1]))

    def upload_host_ptrs(self, n: int, nnz: int, indptr_ptr: int, indices_ptr: int, values_ptr: int = 0,
                         validate: bool = False) -> Subgraph:
        out = _vp()
        check(gsg_subgraph_upload(self.h, n, nnz, indptr_ptr, indices_ptr or None, values_ptr or None, int(validate),
                                  ctypes.byref(out)))
        return Subgraph(self, out.value, n, nnz)

    def upload_device(self, d_indptr, d_indices, d_values=None) -> Subgraph:
        n = d_indptr.numel() - 1
        nnz = d_indices.numel()
        out = _vp()
        check(gsg_subgraph_upload_device(self.h, n, nnz, _ptr(d_indptr), _ptr(d_indices) or None,
                                         _ptr(d_values) or None, ctypes.byref(out)))
        return Subgraph(self, out.value, n, nnz)

    def create_device(self, n: int, nnz_cap: int) -> Subgraph:
        """gsg_subgraph_create_device: n nodes, room for nnz_cap raw entries; sizes on the device."""
        out = _vp()
        check(gsg_subgraph_create_device(self.h, n, nnz_cap, ctypes.byref(out)))
        return Subgraph(self, out.value, n, nnz_cap)

    # ---- kernels ----
    def gather_rows(self, src, idx_ptr: int, dst, rows: int):
        """dst[r, :] = src[idx[r], :] for r < rows (2-D row-major device tensors of one dtype;
        idx_ptr: device int32 array, e.g. the d_nodes of a GPU sample)."""
        es = src.element_size()
        assert dst.element_size() == es and src.shape[1] == dst.shape[1]
        check(gsg_gather_rows(self.h, rows, src.shape[1] * es, _ptr(src), src.stride(0) * es, idx_ptr, _ptr(dst),
                              dst.stride(0) * es))

    def diag_gather_ceiling(self, X, row_floats: int | None = None) -> float:
        """Random-row-gather GB/s from the device matrix X (gsg_diag_gather_ceiling): the measured
        ceiling of the aggregation kernels when X is L2-resident. Synchronizes the stream."""
        rf = min(256, X.shape[1]) if row_floats is None else row_floats
        out = ctypes.c_double(0.0)
        check(gsg_diag_gather_ceiling(self.h, _ptr(X), X.shape[0], _ld(X), rf, ctypes.byref(out)))
        return out.value

    def spmm(self, sg: Subgraph, X, Y, transpose: bool = False, Ylp=None, mask=None, f: int | None = None,
             mask_bits=None):
        """mask_bits: ReLU bitmask (int32 tensor, n x ceil(f/32) words, see relu_bits) of the gate."""
        f = X.shape[1] if f is None else f
        check(gsg_spmm(self.h, sg.h, int(transpose), f, _ptr(X), _ld(X), _ptr(Y), _ld(Y), _ptr(Ylp) or None, _ld(Ylp),
                       _ptr(mask) or None, _ld(mask), _ptr(mask_bits) or None, _ld(mask_bits)))

    def gemm(self, A, B, C, transA=False, transB=False, precision=GSG_PREC_TF32, epilogue=GSG_EPI_NONE, aux=None,
             Clp=None, split_k=0, accumulate=False, M=None, N=None, K=None, aux_bits=None, C_bits=None):
        M = C.shape[0] if M is None else M
        N = C.shape[1] if N is None else N
        if K is None:
            K = A.shape[0] if transA else A.shape[1]
        check(gsg_gemm(self.h, M, N, K, _ptr(A), _ld(A), int(transA), _ptr(B), _ld(B), int(transB), _ptr(C), _ld(C),
                       _ptr(Clp) or None, _ld(Clp), precision, epilogue, _ptr(aux) or None, _ld(aux),
                       _ptr(aux_bits) or None, _ld(aux_bits), _ptr(C_bits) or None, _ld(C_bits), split_k,
                       int(accumulate)))

    def to_bf16(self, src, dst, rows=None, cols=None):
        rows = src.shape[0] if rows is None else rows
        cols = src.shape[1] if cols is None else cols
        check(gsg_to_bf16(self.h, rows, cols, _ptr(src), _ld(src), _ptr(dst), _ld(dst)))

    def layer_forward(self, sg: Subgraph, X, W, P, H, f_in: int, f_out: int, precision=GSG_PREC_TF32, Plp=None,
                      Hlp=None, flags: int = 0, H_bits=None):
        check(gsg_layer_forward(self.h, sg.h, f_in, f_out, _ptr(X), _ld(X), _ptr(W), _ld(W), _ptr(P), _ld(P),
                                _ptr(Plp) or None, _ld(Plp), _ptr(H), _ld(H), _ptr(Hlp) or None, _ld(Hlp),
                                _ptr(H_bits) or None, _ld(H_bits), precision, flags))

    def layer_backward(self, sg: Subgraph, P, H, dH, W, dW, dX, f_in: int, f_out: int, precision=GSG_PREC_TF32,
                       Plp=None, dHlp=None, dXlp=None, H_below=None, flags: int = 0, H_below_bits=None):
        check(gsg_layer_backward(self.h, sg.h, f_in, f_out, _ptr(P), _ld(P), _ptr(Plp) or None, _ld(Plp),
                                 _ptr(H) or None, _ld(H), _ptr(dH), _ld(dH), _ptr(dHlp) or None, _ld(dHlp),
                                 _ptr(W), _ld(W), _ptr(dW), _ld(dW), _ptr(dX) or None, _ld(dX), _ptr(dXlp) or None,
                                 _ld(dXlp), _ptr(H_below) or None, _ld(H_below), _ptr(H_below_bits) or None,
                                 _ld(H_below_bits), precision, flags))

    def sage_forward(self, sg: Subgraph, X, Ws, Wn, P, H, f_in: int, f_half: int, precision=GSG_PREC_TF32,
                     flags: int = 0):
        check(gsg_sage_forward(self.h, sg.h, f_in, f_half, _ptr(X), _ld(X), _ptr(Ws), _ld(Ws), _ptr(Wn), _ld(Wn),
                               _ptr(P), _ld(P), _ptr(H), _ld(H), precision, flags))

    def sage_backward(self, sg: Subgraph, X, P, H, dH, Ws, Wn, dWs, dWn, dX, f_in: int, f_half: int, H_below=None,
                      precision=GSG_PREC_TF32, flags: int = 0):
        check(gsg_sage_backward(self.h, sg.h, f_in, f_half, _ptr(X), _ld(X), _ptr(P), _ld(P), _ptr(H) or None, _ld(H),
                                _ptr(dH), _ld(dH), _ptr(Ws), _ld(Ws), _ptr(Wn), _ld(Wn), _ptr(dWs), _ld(dWs),
                                _ptr(dWn), _ld(dWn), _ptr(dX) or None, _ld(dX), _ptr(H_below) or None, _ld(H_below),
                                precision, flags))

    def head(self, HL, Wm, labels, S, dS, dWm, dHL, n: int, f: int, C: int, kind: int, loss, dHlp=None,
             precision=GSG_PREC_TF32, node_w=None, HL_bits=None):
        check(gsg_head(self.h, n, f, C, kind, _ptr(HL), _ld(HL), _ptr(Wm), _ld(Wm), _ptr(labels), _ptr(S), _ptr(dS),
                       _ld(S), _ptr(dWm), _ld(dWm), _ptr(dHL), _ld(dHL), _ptr(dHlp) or None, _ld(dHlp), _ptr(loss),
                       precision, _ptr(node_w) or None, _ptr(HL_bits) or None, _ld(HL_bits)))

    # ---- data parallel ----
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(gsg_nccl_unique_id(buf))
        return buf.raw

    def nccl_comm_init(self, nranks: int, rank: int, uid: bytes) -> int:
        out = _vp()
        buf = ctypes.create_string_buffer(uid, 128)
        check(gsg_nccl_comm_init(self.h, nranks, rank, buf, ctypes.byref(out)))
        return out.value

    @staticmethod
    def nccl_comm_destroy(comm: int):
        check(gsg_nccl_comm_destroy(comm))

    def wait_event(self, event):
        """Context stream waits for a torch.cuda.Event (an external-event node when capturing)."""
        check(gsg_ctx_wait_event(self.h, event.cuda_event))

    def nccl_wait(self, comm: int, timeout_ms: int = 300000):
        """Wait for this context's stream with NCCL failure detection (gsg_nccl_wait): raises
        GsgError (and aborts the communicator) on an asynchronous NCCL error or a timeout."""
        check(gsg_nccl_wait(self.h, comm, int(timeout_ms)))

    def allreduce_grads(self, comm: int, tensors, average: bool = True):
        n = len(tensors)
        bufs = (_vp * n)(*[_ptr(t) for t in tensors])
        counts = (_i64 * n)(*[t.numel() for t in tensors])
        check(gsg_allreduce_grads(self.h, comm, bufs, counts, n, int(average)))
