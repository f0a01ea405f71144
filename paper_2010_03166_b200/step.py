"""One data-parallel training step of an L-layer GCN on a sampled subgraph, composed only of
C-ABI calls (every row of SURVEY §8(a)):

  a1  gsg_subgraph_normalize                      Â, Âᵀ values, degree bins
  a2  gsg_layer_forward: P = Â X                  (fp32 SpMM)
  a3                     H = ReLU(P W)            (tcgen05 GEMM, fused ReLU)
  a8  gsg_head           S, CE loss, dS, dW_mlp, dH_L = (dS W_mlpᵀ) ⊙ 1[H_L > 0]
  a4-a7 gsg_layer_backward (top down):  dW = Pᵀ dZ ; T = dZ Wᵀ ; dX = Âᵀ T ⊙ 1[H_below > 0]
  a9  gsg_allreduce_grads                         NCCL mean of all dW (one flat buffer)

This mirrors Alg. 1 lines 3-13 minus the weight update, for the GCN model
of Eq. 5 with the backward of P:719. Buffers are allocated once for the largest
subgraph; the step itself allocates nothing (CUDA-graph friendly).
"""
from __future__ import annotations

import os

import torch

from . import (GSG_DH_PREMASKED, GSG_H_BITS, GSG_HEAD_SIGMOID, GSG_HEAD_SOFTMAX, GSG_NORM_ROW_SELF, GSG_ORDER_A_XW,
               GSG_PREC_BF16, GSG_PREC_FP32X3, GSG_PREC_TF32, GSG_W_BF16, Context, Subgraph)


def chain_order(f_in: int, f_out: int) -> int:
    """§7.1: (Â X) W costs δn²·f_in + n·f_in·f_out MACs, Â (X W) costs δn²·f_out +
    n·f_in·f_out; order 2 iff f_in > f_out. Ties keep order 1 (equal MACs; the north star's order)."""
    return 2 if f_in > f_out else 1


def spmm_widths(dims, order, input_grad: bool = True) -> list:
    """Feature widths of the aggregation launches of one step, in launch order: the forward's
    a2 per layer (f_in under order 1, f_out under order 2), then the backward's a7 from the top
    layer down (layer 1's a7 is skipped without the input gradient under order 1)."""
    L = len(dims) - 1
    w = [dims[l + 1] if order[l] == 2 else dims[l] for l in range(L)]
    back = [w[l] for l in range(L - 1, -1, -1) if l > 0 or input_grad or order[l] == 2]
    return w + back


def ld_for(f: int, align: int = 8) -> int:
    return (f + align - 1) // align * align


def padded(rows: int, f: int, dtype=torch.float32, align: int = 8, device="cuda"):
    """Row-major [rows x f] view of a [rows x ld] buffer (ld multiple of 8 elements)."""
    return torch.zeros((rows, ld_for(f, align)), dtype=dtype, device=device)[:, :f]


class GCNStep:
    def __init__(self, ctx: Context, dims: list, n_max: int, head: str = "none", classes: int = 0,
                 precision: str = "tf32", device: int = 0, weights=None, w_mlp=None, order: str = "auto",
                 relu_bits: bool = True):
        self.ctx, self.dims, self.n_max = ctx, list(dims), n_max
        self.L = len(dims) - 1
        self.order = [chain_order(dims[l], dims[l + 1]) if order == "auto" else int(order) for l in range(self.L)]
        self.head = head
        self.C = classes
        self.prec = {"bf16": GSG_PREC_BF16, "fp32x3": GSG_PREC_FP32X3, "tf32": GSG_PREC_TF32}[precision]
        dev = torch.device("cuda", device)
        bf = self.prec == GSG_PREC_BF16
        # weights of equal output width (config 4: 200 -> 1024 x 4) are row blocks of one buffer, so
        # that the per-step bf16 copy of all of them is ONE gsg_to_bf16 call, not one per layer
        ldw = {ld_for(dims[l + 1]) for l in range(self.L)}
        self._w_flat = None
        if len(ldw) == 1 and len({dims[l + 1] for l in range(self.L)}) == 1:
            ld, rows = ldw.pop(), sum(dims[:self.L])
            self._w_flat = torch.zeros((rows, ld), dtype=torch.float32, device=dev)[:, :dims[1]]
            self._wlp_flat = (torch.zeros((rows, ld_for(dims[1], 8)), dtype=torch.bfloat16, device=dev)[:, :dims[1]]
                              if bf else None)
            offs = [sum(dims[:l]) for l in range(self.L + 1)]
            self.W = [self._w_flat[offs[l]:offs[l + 1]] for l in range(self.L)]
        else:
            self.W = [padded(dims[l], dims[l + 1], device=dev) for l in range(self.L)]
        if weights is not None:
            for w, src in zip(self.W, weights):
                w.copy_(torch.as_tensor(src))
        # order 1 keeps P = Â X (n x f_in); order 2 keeps Y = X W (n x f_out) in the same slot
        self.P = [padded(n_max, dims[l + 1] if self.order[l] == 2 else dims[l], device=dev) for l in range(self.L)]
        self.H = [padded(n_max, dims[l + 1], device=dev) for l in range(self.L)]
        self.dX = [padded(n_max, dims[l], device=dev) for l in range(self.L)]
        self.Plp = [padded(n_max, dims[l], torch.bfloat16, device=dev) if bf else None for l in range(self.L)]
        # bf16 weight copies, converted once per step and shared by each layer's forward and
        # backward GEMMs (GSG_W_BF16) instead of one conversion per GEMM call
        if self._w_flat is not None and bf:
            self.Wlp = [self._wlp_flat[offs[l]:offs[l + 1]] for l in range(self.L)]
        else:
            self.Wlp = [padded(dims[l], dims[l + 1], torch.bfloat16, device=dev) if bf else None for l in range(self.L)]
        # (layer 1's dX has no consumer below it: no bf16 copy)
        self.dXlp = [padded(n_max, dims[l], torch.bfloat16, device=dev) if bf and l > 0 else None for l in range(self.L)]
        # ReLU bitmasks of H (gsg.h): the forward epilogue writes 1[H > 0] as bits and the
        # backward gates (SpMMᵀ of the layer above, the head's dH_L GEMM) read 1/32 of the bytes
        # (without a head the top layer's bits gate its own dZ = dH ⊙ 1[H > 0] (GSG_H_BITS) where H is
        # large enough for the saved bytes to matter: config 4 k_mask 33.2 -> 21.6 us, step 1.906 ->
        # 1.891 ms, batched config 1 (x64) 0.447 -> 0.434 ms; on config 1's single 2000 x 128 layer
        # writing and reading the bits costs ~1 us more than it saves)
        top_bits = os.environ.get("GSG_STEP_TOP_BITS", "1") != "0"  # A/B
        self.Hb = [torch.zeros((n_max, (dims[l + 1] + 31) // 32), dtype=torch.int32, device=dev)
                   if relu_bits and (l < self.L - 1 or head != "none" or (top_bits and n_max * dims[l + 1] >= (1 << 21)))
                   else None
                   for l in range(self.L)]
        # all weight gradients in one flat buffer -> one allreduce (a9)
        # (rows padded to 16-byte strides; the padding is reduced along harmlessly)
        shapes = [(dims[l], dims[l + 1]) for l in range(self.L)]
        if head != "none":
            shapes.append((dims[-1], classes))
        sizes = [r * ld_for(c, 4) for r, c in shapes]
        self.grad_flat = torch.zeros(sum(sizes), dtype=torch.float32, device=dev)
        views, off = [], 0
        for (r, c), s in zip(shapes, sizes):
            views.append(self.grad_flat[off:off + s].view(r, ld_for(c, 4))[:, :c])
            off += s
        self.dW = views[:self.L]
        if head != "none":
            self.Wm = padded(dims[-1], classes, device=dev)
            if w_mlp is not None:
                self.Wm.copy_(torch.as_tensor(w_mlp))
            self.dWm = views[self.L]
            self.S = padded(n_max, classes, device=dev)
            self.dS = torch.zeros((n_max, self.S.stride(0)), device=dev)[:, :classes]
            self.dHL = padded(n_max, dims[-1], device=dev)
            self.dHLlp = padded(n_max, dims[-1], torch.bfloat16, device=dev) if bf else None
        self.loss = torch.zeros(1, dtype=torch.float32, device=dev)

    def forward_backward(self, sg: Subgraph, X, labels=None, dH_top=None, comm=None, normalize: bool = True,
                         before_grads=None, input_grad: bool = True, node_w=None):
        """One step. `before_grads` (optional) is called right before the first write of a weight
        gradient (the head, else the top layer's backward): bench.py uses it to make the step
        wait for the previous step's all-reduce of the same gradient buffer, so that the
        all-reduce overlaps this step's forward. `input_grad=False` skips layer 1's dX (the
        gradient w.r.t. the input features, which training does not use). `node_w`
        (optional, device fp32 [n]) are the head's per-node loss weights (gsg_head), e.g. 1/n_k
        and 0 for the padding nodes of a gsg_sample_load subgraph."""
        ctx, d, n = self.ctx, self.dims, sg.n
        if normalize:
            sg.normalize(GSG_NORM_ROW_SELF)
        bf = self.prec == GSG_PREC_BF16
        if bf and self._w_flat is not None:
            ctx.to_bf16(self._w_flat, self._wlp_flat)
        elif bf:
            for w, wl in zip(self.W, self.Wlp):
                ctx.to_bf16(w, wl)
        Wop = self.Wlp if bf else self.W
        wflag = GSG_W_BF16 if bf else 0
        h = X
        inputs = []
        for l in range(self.L):
            inputs.append(h)
            o2 = self.order[l] == 2
            ctx.layer_forward(sg, h, Wop[l], self.P[l][:n], self.H[l][:n], d[l], d[l + 1], precision=self.prec,
                              Plp=None if (self.Plp[l] is None or o2) else self.Plp[l][:n],
                              flags=(GSG_ORDER_A_XW if o2 else 0) | wflag, H_bits=self._hb(l, n))
            h = self.H[l][:n]
        if before_grads is not None:
            before_grads()
        if self.head != "none":
            kind = GSG_HEAD_SOFTMAX if self.head == "softmax" else GSG_HEAD_SIGMOID
            ctx.head(h, self.Wm, labels, self.S[:n], self.dS[:n], self.dWm, self.dHL[:n], n, d[-1], self.C, kind,
                     self.loss, dHlp=None if self.dHLlp is None else self.dHLlp[:n], precision=self.prec,
                     node_w=node_w, HL_bits=self._hb(self.L - 1, n))
            dH, dHlp, flags = self.dHL[:n], (None if self.dHLlp is None else self.dHLlp[:n]), GSG_DH_PREMASKED
        else:  # the caller's dH: the top layer's backward gates it, from H's bitmask when there is one
            dH, dHlp, flags = dH_top, None, (GSG_H_BITS if self.Hb[-1] is not None else 0)
        for l in range(self.L - 1, -1, -1):
            Hbits = self._hb(l - 1, n) if l > 0 else None
            Hb = self.H[l - 1][:n] if l > 0 and Hbits is None else None
            o2 = self.order[l] == 2
            Pl = inputs[l] if o2 else self.P[l][:n]   # order 2 differentiates through X W: needs X
            Plp = None if self.Plp[l] is None else self.Plp[l][:n]
            if o2 and Plp is not None:
                ctx.to_bf16(inputs[l], Plp)
            dXl = self.dX[l][:n] if (l > 0 or input_grad) else None
            Hown = self._hb(l, n) if flags & GSG_H_BITS else self.H[l][:n]
            ctx.layer_backward(sg, Pl, Hown, dH, Wop[l], self.dW[l], dXl,
                               d[l], d[l + 1], precision=self.prec, Plp=Plp, dHlp=dHlp,
                               dXlp=None if (self.dXlp[l] is None or l == 0) else self.dXlp[l][:n], H_below=Hb,
                               flags=flags | (GSG_ORDER_A_XW if o2 else 0) | wflag, H_below_bits=Hbits)
            dH = self.dX[l][:n]
            dHlp = None if self.dXlp[l] is None else self.dXlp[l][:n]
            flags = GSG_DH_PREMASKED  # the transposed aggregation already applied layer l-1's ReLU' gate
        if comm is not None:
            ctx.allreduce_grads(comm, [self.grad_flat], average=True)
        return self.loss

    def _hb(self, l: int, n: int):
        return None if self.Hb[l] is None else self.Hb[l][:n]

    def spmm_widths(self, input_grad: bool = True) -> list:
        return spmm_widths(self.dims, self.order, input_grad)

    def work_edge_features(self, nnz_hat: int, input_grad: bool = True) -> int:
        """2 * nnz' * f edge-features per layer (a2 + a7), summed over layers, where f is
        the width the aggregation runs at: f_in under order 1, f_out under order 2. Without the
        input gradient, layer 1's a7 is not run under order 1 (under order 2 its G = Âᵀ dZ still
        feeds dW)."""
        w = sum(2 * nnz_hat * (self.dims[l + 1] if self.order[l] == 2 else self.dims[l]) for l in range(self.L))
        if not input_grad and self.order[0] == 1:
            w -= nnz_hat * self.dims[0]
        return w

    def gemm_flops(self, n: int) -> int:
        f = 6 * sum(n * self.dims[l] * self.dims[l + 1] for l in range(self.L))
        if self.head != "none":
            f += 6 * n * self.dims[-1] * self.C
        return f
