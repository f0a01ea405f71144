"""Host workload generator: determinism, CSR invariants, induction.

Pins: induction equals a brute-force double loop over node pairs; the
frontier sampler returns exactly n distinct nodes (Alg. 2, "until the size of V_s
reaches the desired budget n", reading R9); clipping yields a multiple of 16.
"""
import numpy as np
import pytest

import workload as wl


def check_csr(csr: wl.CSR):
    ip, ix = csr.indptr, csr.indices
    n = csr.n
    assert ip[0] == 0 and np.all(np.diff(ip) >= 0)
    assert ix.size == ip[-1]
    if ix.size:
        assert ix.min() >= 0 and ix.max() < n
    rows = np.repeat(np.arange(n), np.diff(ip))
    assert not np.any(rows == ix), "self loop"
    for i in range(n):
        r = ix[ip[i]:ip[i + 1]]
        assert np.all(np.diff(r) > 0), "rows must be strictly ascending (no duplicates)"
    # symmetry: the multiset of (i,j) equals that of (j,i)
    a = rows.astype(np.int64) * n + ix
    b = ix.astype(np.int64) * n + rows
    assert np.array_equal(np.sort(a), np.sort(b))


def test_parent_invariants_and_determinism():
    p1 = wl.Parent(3000, 12.0, 2.1, 0.0, seed=7).csr()
    p2 = wl.Parent(3000, 12.0, 2.1, 0.0, seed=7).csr()
    p3 = wl.Parent(3000, 12.0, 2.1, 0.0, seed=8).csr()
    check_csr(p1)
    assert np.array_equal(p1.indptr, p2.indptr) and np.array_equal(p1.indices, p2.indices)
    assert not np.array_equal(p1.indices[:100], p3.indices[:100])
    mean = p1.nnz / p1.n
    assert 0.98 * 12.0 <= mean < 1.3 * 12.0
    # heavy tail: max degree well above the mean (power law, gamma 2.1)
    assert p1.degrees().max() > 5 * mean


def test_frontier_sample_budget_and_clip():
    p = wl.Parent(5000, 10.0, 2.1, 0.0, seed=3)
    s = p.frontier_sample(n=1008, m=100, seed=11, clip=16)
    check_csr(s)
    assert s.n == 1008  # already a multiple of 16 -> no-op clip
    assert np.all(np.diff(s.nodes) > 0)
    s2 = p.frontier_sample(n=1008, m=100, seed=11, clip=16)
    assert np.array_equal(s.indices, s2.indices)
    s3 = p.frontier_sample(n=1001, m=100, seed=12, clip=16)
    assert s3.n == 992  # clipped down to a multiple of 16


def test_induction_equals_bruteforce():
    p = wl.Parent(200, 6.0, 2.1, 0.0, seed=5)
    pc = p.csr()
    rng = np.random.default_rng(0)
    nodes = np.sort(rng.choice(200, 50, replace=False))
    sub = p.induce(nodes)
    check_csr(sub)
    adj = set()
    for i in range(pc.n):
        for j in pc.indices[pc.indptr[i]:pc.indptr[i + 1]]:
            adj.add((i, int(j)))
    expect = []
    for a, u in enumerate(nodes):
        for b, v in enumerate(nodes):
            if (int(u), int(v)) in adj:
                expect.append((a, b))
    got = [(i, int(j)) for i in range(sub.n) for j in sub.indices[sub.indptr[i]:sub.indptr[i + 1]]]
    assert got == expect


def test_full_induction_is_identity():
    p = wl.Parent(300, 5.0, 2.1, 0.0, seed=9)
    pc = p.csr()
    sub = p.induce(np.arange(300))
    assert np.array_equal(sub.indptr, pc.indptr) and np.array_equal(sub.indices, pc.indices)


def test_inputs_seeded():
    cfg = wl.tiny_config(head="sigmoid", classes=7)
    a = wl.make_inputs(cfg, 64)
    b = wl.make_inputs(cfg, 64)
    c = wl.make_inputs(cfg, 64, r=1)
    assert np.array_equal(a.X, b.X) and not np.array_equal(a.X, c.X)
    assert np.array_equal(a.Ws[0], c.Ws[0])  # weights replicated across ranks
    lim = np.sqrt(6.0 / (cfg.dims[0] + cfg.dims[1]))
    assert np.abs(a.Ws[0]).max() <= lim
    assert a.labels.shape == (64, 7) and a.labels.dtype == np.uint8


@pytest.mark.parametrize("cid", [1, 2])
def test_config_shapes(cid):
    cfg = wl.CONFIGS[cid]
    s = wl.sample_subgraph(cfg)
    check_csr(s)
    assert s.n == cfg.n
    st = s.stats()
    if cid == 2:  # SURVEY Appendix A calibration: stated ~200K nnz (±15%)
        assert 170_000 <= st["nnz"] <= 230_000


def test_block_diag_batch_structure():
    """block_diag: disjoint union (config-1 batched variant): sizes add up, every
    part keeps its own edges (shifted), no edge crosses parts, symmetry is preserved."""
    cfg = wl.tiny_config(n_parent=300, mean_deg=6.0, n=40, m=8)
    parts = [wl.sample_subgraph(cfg, k) for k in range(3)]
    g = wl.block_diag(parts)
    assert g.n == sum(p.n for p in parts) and g.nnz == sum(p.nnz for p in parts)
    off = 0
    for p in parts:
        for i in range(p.n):
            row = g.indices[g.indptr[off + i]:g.indptr[off + i + 1]]
            assert np.array_equal(row, p.indices[p.indptr[i]:p.indptr[i + 1]] + off)
        off += p.n
    A = np.zeros((g.n, g.n), np.int8)
    for i in range(g.n):
        A[i, g.indices[g.indptr[i]:g.indptr[i + 1]]] = 1
    assert np.array_equal(A, A.T)
    b = wl.sample_batch(cfg, 3)
    assert np.array_equal(b.indptr, g.indptr) and np.array_equal(b.indices, g.indices)
