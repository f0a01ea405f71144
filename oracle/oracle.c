/* oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the GCN-layer hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2010_03166_b200/, libgsg.so) never links, loads or calls it, and this file shares
 * no code, header, table or constant with the CUDA path.
 *
 * Every function computes the plain definition it cites (SURVEY §8(c) "Oracle"):
 *   - normalized adjacency:   Eq. 5, row mode D~^-1 (A+I),
 *                             GraphSAGE D^-1 A (Eq. 1)
 *   - transpose data array:   Alg. 4, serial, verbatim
 *   - feature aggregation:    P = Â X, row loops (Alg. 6's product)
 *   - transposed aggregation: dX = Âᵀ T in SCATTER form from the definition of the transpose:
 *                             every stored (i, j, a) adds a*T[i,:] to dX[j,:] (never uses Alg. 4)
 *   - dense products:         C = op(A) op(B), triple loops (weight transformation)
 *   - loss head:              Eqs. 2-4 forward and Eqs. 9-11 backward
 * All arithmetic is double precision; inputs arrive as double (the Python wrapper upcasts).
 * OpenMP is used only over independent output rows (or independent output column slabs for
 * the scatter, i.e. Alg. 6's feature-only partitioning), which does not change
 * any individual sum's order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_NORM_ROW_SELF 0 /* D~^-1 (A+I), D~ = D + I: the configs            */
#define OR_NORM_SYM_SELF 1 /* (I+D)^-1/2 (I+A) (I+D)^-1/2: Eq. 5            */
#define OR_NORM_ROW      2 /* D^-1 A: GraphSAGE Eq. 1, PAPER.md:131 (isolated rows = 0)    */
#define OR_NORM_VALUES   3 /* Â_ij = given values, no self loop (weighted Â)    */

/* Number of stored entries of Â for a binary CSR with nnz entries (self loops added in
 * the *_SELF modes). */
int64_t oracle_nnz_hat(int32_t n, int64_t nnz, int mode) {
  return (mode == OR_NORM_ROW_SELF || mode == OR_NORM_SYM_SELF) ? nnz + n : nnz;
}

/* Build Â in CSR: for each row i the entries are (i, j) for j in N(i) (plus i itself in the
 * *_SELF modes, inserted at its sorted position); values per the mode's definition. The
 * degree d_i = |N_s(i)| is subgraph-local. */
void oracle_normalize(int32_t n, const int64_t* indptr, const int32_t* indices,
                      const double* values, int mode,
                      int64_t* indptr_h, int32_t* idx_h, double* val_h) {
  int self = (mode == OR_NORM_ROW_SELF || mode == OR_NORM_SYM_SELF);
  indptr_h[0] = 0;
  for (int32_t i = 0; i < n; i++) indptr_h[i + 1] = indptr_h[i] + (indptr[i + 1] - indptr[i]) + self;
  for (int32_t i = 0; i < n; i++) {
    int64_t o = indptr_h[i];
    int inserted = !self;
    double di = (double)(indptr[i + 1] - indptr[i]);
    for (int64_t k = indptr[i]; k <= indptr[i + 1]; k++) {
      if (!inserted && (k == indptr[i + 1] || indices[k] > i)) {
        idx_h[o] = i;
        val_h[o] = (mode == OR_NORM_ROW_SELF) ? 1.0 / (di + 1.0) : 1.0 / sqrt((di + 1.0) * (di + 1.0));
        o++;
        inserted = 1;
      }
      if (k == indptr[i + 1]) break;
      int32_t j = indices[k];
      double dj = (double)(indptr[j + 1] - indptr[j]);
      double a;
      switch (mode) {
        case OR_NORM_ROW_SELF: a = 1.0 / (di + 1.0); break;
        case OR_NORM_SYM_SELF: a = 1.0 / sqrt((di + 1.0) * (dj + 1.0)); break;
        case OR_NORM_ROW: a = 1.0 / di; break;
        default: a = values[k]; break;
      }
      idx_h[o] = j;
      val_h[o] = a;
      o++;
    }
  }
}

/* Alg. 4, verbatim: one serial pass over Indptr/Indices appending each
 * a = Data[j] of edge (v, u) to row u's slice of DataTrans. Requires ascending rows and a
 * symmetric structure. Returns 0, or -1 if a row overflows (asymmetry). */
int oracle_transpose_alg4(int32_t n, const int64_t* indptr, const int32_t* indices,
                          const double* data, double* data_trans) {
  int64_t* ptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int32_t v = 0; v < n; v++) ptr[v] = indptr[v];          /* PtrData <- Indptr[:|V_s|] */
  int rc = 0;
  for (int32_t v = 0; v < n && rc == 0; v++) {
    for (int64_t j = indptr[v]; j < indptr[v + 1]; j++) {
      int32_t u = indices[j];
      double a = data[j];
      if (ptr[u] >= indptr[u + 1]) { rc = -1; break; }
      data_trans[ptr[u]] = a;                                    /* DataTrans[PtrData[u]] <- a */
      ptr[u]++;                                                  /* next position to append   */
    }
  }
  free(ptr);
  return rc;
}

/* P[i,:] = sum_{k in row i} Â_ik X[idx_k,:]  for rows i in [r0, r1). X is n x f (ld ldx),
 * P is written at rows r0..r1-1 (ld ldp). */
void oracle_spmm(int32_t n, int32_t f, const int64_t* indptr, const int32_t* idx, const double* val,
                 const double* X, int64_t ldx, int32_t r0, int32_t r1, double* P, int64_t ldp) {
  (void)n;
#pragma omp parallel for schedule(dynamic, 16)
  for (int32_t i = r0; i < r1; i++) {
    double* p = P + (int64_t)i * ldp;
    for (int32_t c = 0; c < f; c++) p[c] = 0.0;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; k++) {
      const double a = val[k];
      const double* x = X + (int64_t)idx[k] * ldx;
      for (int32_t c = 0; c < f; c++) p[c] += a * x[c];
    }
  }
}

/* dX = Âᵀ T restricted to the contributions of source rows i in [r0, r1), in scatter form
 * from the definition of the transpose: for every stored (i, j, a) of Â, dX[j,:] += a*T[i,:].
 * dX (n x f, ld lddx) is zeroed first. Columns are split into independent slabs across
 * threads (Alg. 6's feature partitioning); within a column the sum order is the serial
 * (i, k) order. */
void oracle_spmm_t_scatter(int32_t n, int32_t f, const int64_t* indptr, const int32_t* idx,
                           const double* val, const double* T, int64_t ldt, int32_t r0, int32_t r1,
                           double* dX, int64_t lddx) {
  for (int32_t j = 0; j < n; j++)
    for (int32_t c = 0; c < f; c++) dX[(int64_t)j * lddx + c] = 0.0;
  const int32_t slab = 32;
  const int32_t nslab = (f + slab - 1) / slab;
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t s = 0; s < nslab; s++) {
    const int32_t c0 = s * slab, c1 = (c0 + slab < f) ? c0 + slab : f;
    for (int32_t i = r0; i < r1; i++) {
      const double* t = T + (int64_t)i * ldt;
      for (int64_t k = indptr[i]; k < indptr[i + 1]; k++) {
        const double a = val[k];
        double* d = dX + (int64_t)idx[k] * lddx;
        for (int32_t c = c0; c < c1; c++) d[c] += a * t[c];
      }
    }
  }
}

/* C[M x N] = op(A) op(B), op(A) = A (M x K, ld lda) or Aᵀ (A stored K x M); same for B.
 * Plain triple loop, one output row per OpenMP iteration. */
void oracle_gemm(int32_t M, int32_t N, int32_t K, const double* A, int64_t lda, int transA,
                 const double* B, int64_t ldb, int transB, double* C, int64_t ldc) {
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < M; i++) {
    double* c = C + (int64_t)i * ldc;
    for (int32_t j = 0; j < N; j++) c[j] = 0.0;
    for (int32_t k = 0; k < K; k++) {
      const double a = transA ? A[(int64_t)k * lda + i] : A[(int64_t)i * lda + k];
      if (!transB) {
        const double* b = B + (int64_t)k * ldb;
        for (int32_t j = 0; j < N; j++) c[j] += a * b[j];
      } else {
        for (int32_t j = 0; j < N; j++) c[j] += a * B[(int64_t)j * ldb + k];
      }
    }
  }
}

/* Classifier head and CE loss (Eqs. 2-4; backward Eqs. 9-10; SURVEY
 * §8(c) step 8, readings R7/R8):
 *   S+ = ReLU(S); Y = softmax_rows(S+) (kind 0) or sigmoid(S+) (kind 1)
 *   kind 0: L = -(1/n) sum_i log Y[i, y_i]                       (labels: int32 class ids)
 *   kind 1: L = (1/n) sum_{i,c} [log(1+e^-|s|) + max(s,0) - ybar*s],  s = S+[i,c]
 *                                                                (labels: uint8 indicator)
 *   dS+ = (Y - Ybar)/n ;  dS = dS+ * 1[S > 0]  (mask of the head's ReLU, R4)
 * With per-node weights w (GraphSAINT loss normalization: "the loss L_s would be
 * computed with weighted sum"), 1/n is replaced by w[i] in both L and dS+; w = NULL means 1/n.
 * Returns the loss; writes Y and dS (n x C, ld C). */
double oracle_head(int32_t n, int32_t C, const double* S, int64_t lds, int kind,
                   const int32_t* cls, const uint8_t* ind, const double* w, double* Y, double* dS) {
  double loss = 0.0;
#pragma omp parallel for reduction(+ : loss) schedule(static)
  for (int32_t i = 0; i < n; i++) {
    const double lam = w ? w[i] : 1.0 / n;
    double li = 0.0;
    const double* s = S + (int64_t)i * lds;
    double* y = Y + (int64_t)i * C;
    double* g = dS + (int64_t)i * C;
    if (kind == 0) {
      double mx = -INFINITY;
      for (int32_t c = 0; c < C; c++) { double sp = s[c] > 0 ? s[c] : 0.0; if (sp > mx) mx = sp; }
      double z = 0.0;
      for (int32_t c = 0; c < C; c++) { double sp = s[c] > 0 ? s[c] : 0.0; z += exp(sp - mx); }
      double lse = mx + log(z);
      for (int32_t c = 0; c < C; c++) {
        double sp = s[c] > 0 ? s[c] : 0.0;
        y[c] = exp(sp - lse);
        double ybar = (c == cls[i]) ? 1.0 : 0.0;
        g[c] = (s[c] > 0) ? lam * (y[c] - ybar) : 0.0;
      }
      double spy = s[cls[i]] > 0 ? s[cls[i]] : 0.0;
      li = -(spy - lse);
    } else {
      for (int32_t c = 0; c < C; c++) {
        double sp = s[c] > 0 ? s[c] : 0.0;
        double ybar = ind[(int64_t)i * C + c] ? 1.0 : 0.0;
        y[c] = 1.0 / (1.0 + exp(-sp));
        li += log1p(exp(-fabs(sp))) + (sp > 0 ? sp : 0.0) - ybar * sp;
        g[c] = (s[c] > 0) ? lam * (y[c] - ybar) : 0.0;
      }
    }
    loss += lam * li;
  }
  return loss;
}

/* ---------------------------------------------------------------------------------------
 * Frontier sampling, Alg. 2 under reading R9, plain and serial, with the
 * counter-based draws specified in include/gsg.h (so the GPU sampler must reproduce it bit for
 * bit):  r(i, j) = mix64(seed ^ mix64(4 i + j)),  below(r, N) = ((r >> 32) * N) >> 32.
 * The frontier pop is written as its definition: scan the frontier in slot order and take the
 * first slot whose cumulative degree exceeds x (x uniform below the total) -- no tree.
 * Writes the ascending node list (n_out nodes) into nodes_out[n]. Returns n_out.
 * --------------------------------------------------------------------------------------- */
static uint64_t or_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t or_rng(uint64_t seed, uint64_t i, uint32_t j) { return or_mix64(seed ^ or_mix64(4 * i + j)); }
static uint32_t or_below(uint64_t r, uint32_t N) { return (uint32_t)(((r >> 32) * (uint64_t)N) >> 32); }
static int or_cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

int32_t oracle_frontier_sample(int64_t N, const int64_t* indptr, const int32_t* indices, int32_t n, int32_t m,
                               int32_t clip, uint64_t seed, int32_t* nodes_out) {
  int32_t* noniso = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);
  int64_t n_noniso = 0;
  for (int64_t v = 0; v < N; v++)
    if (indptr[v + 1] > indptr[v]) noniso[n_noniso++] = (int32_t)v;
  unsigned char* in_vs = (unsigned char*)calloc((size_t)N, 1);
  int32_t* fs = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
  int32_t* vs = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  /* Alg. 2 line 1 (R9): m distinct non-isolated nodes, uniform; line 2: V_s <- FS */
  int32_t cnt = 0;
  for (uint64_t t = 0; cnt < m; t++) {
    int32_t c = noniso[or_below(or_rng(seed, t, 3), (uint32_t)n_noniso)];
    if (in_vs[c]) continue;
    in_vs[c] = 1;
    fs[cnt] = c;
    vs[cnt] = c;
    cnt++;
  }
  int32_t nv = m;
  const uint64_t max_it = 1000ull * (uint64_t)n + 1000000ull;
  for (uint64_t it = 0; nv < n && it < max_it; it++) {
    int64_t total = 0;
    for (int32_t i = 0; i < m; i++) total += indptr[fs[i] + 1] - indptr[fs[i]];
    /* line 4: select u in FS with probability deg(u) / sum_FS deg */
    int64_t x = or_below(or_rng(seed, it, 0), (uint32_t)total);
    int32_t slot = 0;
    int64_t cum = 0;
    for (slot = 0; slot < m; slot++) {
      cum += indptr[fs[slot] + 1] - indptr[fs[slot]];
      if (cum > x) break;
    }
    int32_t u = fs[slot];
    int64_t du = indptr[u + 1] - indptr[u];
    /* line 5: u' uniformly among the neighbors of u */
    int32_t up = indices[indptr[u] + or_below(or_rng(seed, it, 1), (uint32_t)du)];
    /* line 6: FS <- (FS \ {u}) U {u'} ; R9: u' joins V_s */
    fs[slot] = up;
    if (!in_vs[up]) {
      in_vs[up] = 1;
      vs[nv++] = up;
    }
  }
  /* clipping: drop uniformly random nodes until |V_s| is a multiple of clip */
  int32_t keep = nv / clip * clip;
  for (uint64_t r = 0; nv > keep; r++) {
    int32_t j = (int32_t)or_below(or_rng(seed, r, 2), (uint32_t)nv);
    vs[j] = vs[nv - 1];
    nv--;
  }
  qsort(vs, (size_t)nv, sizeof(int32_t), or_cmp_i32);
  memcpy(nodes_out, vs, sizeof(int32_t) * (size_t)nv);
  free(noniso); free(in_vs); free(fs); free(vs);
  return nv;
}

/* Induced subgraph on an ascending node list (Alg. 2 line 9): local id = position in the list;
 * row i holds the local ids of the neighbors of nodes[i] that are in the list, in the parent's
 * (ascending) order. Two calls: indices_out = NULL returns nnz and fills indptr_out. */
int64_t oracle_induce(int64_t N, const int64_t* indptr, const int32_t* indices, int32_t n, const int32_t* nodes,
                      int64_t* indptr_out, int32_t* indices_out) {
  int32_t* local = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);
  for (int64_t v = 0; v < N; v++) local[v] = -1;
  for (int32_t i = 0; i < n; i++) local[nodes[i]] = i;
  indptr_out[0] = 0;
  for (int32_t i = 0; i < n; i++) {
    int64_t c = 0;
    for (int64_t k = indptr[nodes[i]]; k < indptr[nodes[i] + 1]; k++) {
      int32_t l = local[indices[k]];
      if (l >= 0) {
        if (indices_out) indices_out[indptr_out[i] + c] = l;
        c++;
      }
    }
    indptr_out[i + 1] = indptr_out[i] + c;
  }
  free(local);
  return indptr_out[n];
}
