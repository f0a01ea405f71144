"""Frontier sampling + induction (Alg. 2, reading R9).

not-gpu: the oracle sampler/inducer against what Alg. 2 and the definition of an induced
subgraph fix (budget, distinctness, FS_0 from non-isolated nodes, reachability, degree bias,
brute-force induction, agreement with the independent workload generator's induction).
gpu: the device sampler (gsg_frontier_sample) reproduces the oracle bit for bit -- same
counter-based draws (include/gsg.h) -- and its output trains through the C ABI.
"""
import os

import numpy as np
import pytest

import oracle as orc
import workload as wl


def parent(n=3000, deg=10.0, seed=1):
    return wl.Parent(n, deg, 2.1, 0.0, seed=seed).csr()


def components(csr):
    lab = -np.ones(csr.n, np.int64)
    c = 0
    for s in range(csr.n):
        if lab[s] >= 0:
            continue
        stack = [s]
        lab[s] = c
        while stack:
            v = stack.pop()
            for w in csr.indices[csr.indptr[v]:csr.indptr[v + 1]]:
                if lab[w] < 0:
                    lab[w] = c
                    stack.append(w)
        c += 1
    return lab


def test_oracle_sampler_budget_distinct_deterministic():
    p = parent()
    v1 = orc.frontier_sample(p.indptr, p.indices, 400, 50, 16, seed=7)
    v2 = orc.frontier_sample(p.indptr, p.indices, 400, 50, 16, seed=7)
    v3 = orc.frontier_sample(p.indptr, p.indices, 400, 50, 16, seed=8)
    assert v1.size == 400 and np.array_equal(v1, v2) and not np.array_equal(v1, v3)
    assert np.all(np.diff(v1) > 0)                      # ascending, distinct
    deg = np.diff(p.indptr)
    assert np.all(deg[v1] > 0)                           # only non-isolated nodes are ever reached
    clipped = orc.frontier_sample(p.indptr, p.indices, 401, 50, 16, seed=7)
    assert clipped.size == 400                           # clip to a multiple of 16


def test_oracle_sampler_m_equals_n_is_uniform_start():
    """With m = n no frontier step runs: V_s is FS_0, m distinct non-isolated nodes."""
    p = parent(500, 6.0, 3)
    v = orc.frontier_sample(p.indptr, p.indices, 40, 40, 1, seed=11)
    assert v.size == 40 and len(set(v.tolist())) == 40


def test_oracle_sampler_stays_in_start_components():
    """Every V_s node is reachable from FS_0 (each new node is a neighbor of a frontier node)."""
    g = wl.CSR(np.array([0, 1, 2, 3, 4, 4], np.int64), np.array([1, 0, 3, 2], np.int32))  # two K2 + isolated
    v = orc.frontier_sample(g.indptr, g.indices, 2, 1, 1, seed=5)
    lab = components(g)
    assert v.size == 2 and lab[v[0]] == lab[v[1]]
    p = parent(2000, 3.0, 4)  # sparse parent: several components
    v = orc.frontier_sample(p.indptr, p.indices, 300, 10, 1, seed=6)
    lab = components(p)
    assert np.unique(lab[v]).size <= 10


def test_oracle_sampler_degree_bias():
    """Frontier sampling is degree-biased (pops ∝ degree): sampled nodes have a higher
    mean degree than the parent's non-isolated nodes (statistical pin)."""
    p = parent(20000, 10.0, 9)
    deg = np.diff(p.indptr)
    v = orc.frontier_sample(p.indptr, p.indices, 3000, 300, 1, seed=12)
    assert deg[v].mean() > 1.5 * deg[deg > 0].mean()


def test_oracle_induce_bruteforce_and_independent_impl():
    p = parent(300, 8.0, 13)
    v = orc.frontier_sample(p.indptr, p.indices, 80, 20, 1, seed=14)
    ip, ix = orc.induce(p.indptr, p.indices, v)
    E = {(int(i), int(j)) for i in range(p.n) for j in p.indices[p.indptr[i]:p.indptr[i + 1]]}
    expect = [(a, b) for a in range(v.size) for b in range(v.size) if (int(v[a]), int(v[b])) in E]
    got = [(i, int(j)) for i in range(v.size) for j in ix[ip[i]:ip[i + 1]]]
    assert got == expect
    w = wl.Parent.from_csr(p).induce(v.astype(np.int64))  # the generator's own (host C++) induction
    assert np.array_equal(w.indptr, ip) and np.array_equal(w.indices, ix)


# ---------------------------------------------------------------- Alg. 2 line 4 pin
# Brute force on a tiny parent: the exact distribution of the sampled node set V_s, computed by
# propagating probability mass through Alg. 2's Markov chain (R9 reading) with the frontier pop
# written as P:377 states it -- u in FS with probability deg(u) / sum_{v in FS} deg(v) -- and
# compared with the oracle's empirical distribution over many seeds (chi-square). A uniform pop
# (or a pop by any other weight) gives a different distribution on this graph; the mutation test
# below builds exactly that mutant from oracle.c and checks that the same test rejects it.
_TINY_EDGES = [(0, 1), (0, 2), (0, 3), (0, 4), (0, 5), (1, 6), (6, 7), (7, 8)]


def _tiny_parent():
    n = 9
    adj = [[] for _ in range(n)]
    for a, b in _TINY_EDGES:
        adj[a].append(b)
        adj[b].append(a)
    indptr = np.zeros(n + 1, np.int64)
    indptr[1:] = np.cumsum([len(a) for a in adj])
    indices = np.array([v for a in adj for v in sorted(a)], np.int32)
    return indptr, indices, [sorted(a) for a in adj]


def _exact_vs_distribution(adj, n_budget, m, pop_weight):
    """P(V_s = S) for Alg. 2 (R9): FS_0 = m distinct non-isolated nodes, ordered, uniform; then
    repeat {pop slot s w.p. pop_weight(FS[s]) / sum; u' uniform neighbor of FS[s]; FS[s] <- u';
    V_s <- V_s ∪ {u'}} until |V_s| = n_budget. Mass propagation over (FS, V_s) states."""
    import itertools
    noniso = [v for v in range(len(adj)) if adj[v]]
    start = list(itertools.permutations(noniso, m))
    cur = {}
    for fs in start:
        key = (fs, frozenset(fs))
        cur[key] = cur.get(key, 0.0) + 1.0 / len(start)
    done = {}
    for _ in range(5000):
        nxt = {}
        for (fs, vs), p in cur.items():
            w = [pop_weight(u) for u in fs]
            tot = float(sum(w))
            for s, u in enumerate(fs):
                for up in adj[u]:
                    q = p * (w[s] / tot) / len(adj[u])
                    nfs = fs[:s] + (up,) + fs[s + 1:]
                    nvs = vs | {up}
                    if len(nvs) == n_budget:
                        k = tuple(sorted(nvs))
                        done[k] = done.get(k, 0.0) + q
                    else:
                        nxt[(nfs, nvs)] = nxt.get((nfs, nvs), 0.0) + q
        cur = nxt
        if sum(cur.values()) < 1e-13:
            break
    assert sum(cur.values()) < 1e-9
    return done


def _chi2_pvalue(samples, dist, n_draws):
    from scipy.stats import chi2
    keys = sorted(dist, key=lambda k: -dist[k])
    obs, exp = [], []
    rest_o, rest_e = 0.0, 0.0
    for k in keys:
        e = dist[k] * n_draws
        if e >= 10:
            obs.append(samples.get(k, 0))
            exp.append(e)
        else:
            rest_o += samples.get(k, 0)
            rest_e += e
    unknown = sum(c for k, c in samples.items() if k not in dist)
    obs.append(rest_o + unknown)
    exp.append(rest_e)
    obs, exp = np.array(obs, float), np.array(exp, float)
    if exp[-1] < 1e-12:
        assert obs[-1] == 0, "the sampler produced a node set the brute force gives probability 0"
        obs, exp = obs[:-1], exp[:-1]
    stat = float(((obs - exp) ** 2 / exp).sum())
    return float(chi2.sf(stat, len(obs) - 1))


def _oracle_histogram(sample_fn, indptr, indices, n_budget, m, draws):
    h = {}
    for s in range(draws):
        v = sample_fn(indptr, indices, n_budget, m, 1, 1000 + s)
        k = tuple(int(x) for x in v)
        h[k] = h.get(k, 0) + 1
    return h


_N_BUDGET, _M, _DRAWS = 5, 2, 30000


def test_oracle_frontier_pop_degree_proportional_bruteforce():
    """Alg. 2 line 4: the oracle's V_s distribution equals the exact Markov-chain
    distribution with degree-proportional pops (chi-square, 30K seeds), and is far from the
    uniform-pop distribution on the same graph."""
    indptr, indices, adj = _tiny_parent()
    deg = [len(a) for a in adj]
    exact = _exact_vs_distribution(adj, _N_BUDGET, _M, lambda u: deg[u])
    uniform = _exact_vs_distribution(adj, _N_BUDGET, _M, lambda u: 1)
    assert abs(sum(exact.values()) - 1.0) < 1e-9
    # the two readings are well separated at this sample size (expected chi-square >> threshold)
    sep = _DRAWS * sum((uniform.get(k, 0.0) - p) ** 2 / p for k, p in exact.items())
    assert sep > 500, sep
    h = _oracle_histogram(orc.frontier_sample, indptr, indices, _N_BUDGET, _M, _DRAWS)
    assert _chi2_pvalue(h, exact, _DRAWS) > 1e-4
    assert _chi2_pvalue(h, uniform, _DRAWS) < 1e-12


def test_oracle_frontier_pop_uniform_mutant_is_rejected(tmp_path):
    """Mutation test: oracle.c rebuilt with the pop weight deg(u) replaced by 1 (a uniform pop)
    fails the brute-force pin above -- the pin demonstrably detects the mutant."""
    import ctypes
    import subprocess
    src = open(os.path.join(os.path.dirname(orc.__file__), "oracle.c")).read()
    pop_total = "total += indptr[fs[i] + 1] - indptr[fs[i]];"
    pop_cum = "cum += indptr[fs[slot] + 1] - indptr[fs[slot]];"
    assert src.count(pop_total) == 1 and src.count(pop_cum) == 1, "pop code moved: update the mutation"
    mut = src.replace(pop_total, "total += 1;").replace(pop_cum, "cum += 1;")
    (tmp_path / "m.c").write_text(mut)
    so = tmp_path / "libm.so"
    subprocess.run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-o", str(so), str(tmp_path / "m.c"),
                    "-lm"], check=True)
    L = ctypes.CDLL(str(so))
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.oracle_frontier_sample.restype = i32
    L.oracle_frontier_sample.argtypes = [i64, vp, vp, i32, i32, i32, ctypes.c_uint64, vp]

    def mutant(ip, ix, n, m, clip, seed):
        out = np.empty(n, np.int32)
        nv = L.oracle_frontier_sample(ip.shape[0] - 1, ip.ctypes.data_as(vp), ix.ctypes.data_as(vp), n, m, clip,
                                      seed, out.ctypes.data_as(vp))
        return out[:nv]

    indptr, indices, adj = _tiny_parent()
    deg = [len(a) for a in adj]
    exact = _exact_vs_distribution(adj, _N_BUDGET, _M, lambda u: deg[u])
    uniform = _exact_vs_distribution(adj, _N_BUDGET, _M, lambda u: 1)
    h = _oracle_histogram(mutant, indptr, indices, _N_BUDGET, _M, _DRAWS)
    assert _chi2_pvalue(h, exact, _DRAWS) < 1e-12      # the degree-proportional pin rejects it
    assert _chi2_pvalue(h, uniform, _DRAWS) > 1e-4     # and it is what it claims to be


# ------------------------------------------------------------------------------ GPU
_M64 = (1 << 64) - 1


def _mix64(z):
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def sampler_seed(seed, k):
    """Seed of sampler k of one gsg_frontier_sample call (include/gsg.h: mix64(mix64(seed) + k))."""
    return _mix64((_mix64(seed) + k) & _M64)


def test_sampler_seeds_are_decorrelated():
    """Consecutive calls do not repeat subgraphs: sampler k of seed S != sampler k-1 of seed S+1
    (with seed + k they were identical)."""
    keys = {sampler_seed(s, k) for s in range(50) for k in range(50)}
    assert len(keys) == 2500
    assert sampler_seed(7, 1) != sampler_seed(8, 0)


@pytest.mark.gpu
@pytest.mark.parametrize("cid", [1, 2, 5])
def test_gpu_sampler_matches_oracle(cid):
    import paper_2010_03166_b200 as gsg
    cfg = wl.CONFIGS[cid]
    p = wl.parent_for(cfg).csr()
    ctx = gsg.Context(0)
    pg = gsg.ParentGraph(ctx, p.indptr, p.indices)
    count = 3
    seed = 1234 + cid
    batch = pg.sample(cfg.n, cfg.m, seed, count=count, clip=16)
    for k in range(count):
        ip, ix, nd = batch.to_host(k)
        v = orc.frontier_sample(p.indptr, p.indices, cfg.n, cfg.m, 16, sampler_seed(seed, k))
        assert np.array_equal(nd, v), f"sample {k}: node sets differ"
        rip, rix = orc.induce(p.indptr, p.indices, v)
        assert np.array_equal(ip, rip) and np.array_equal(ix, rix), f"sample {k}: induced CSR differs"
    batch.free()
    pg.free()


@pytest.mark.gpu
def test_gpu_sample_trains():
    """A GPU-sampled subgraph feeds the layer path directly (device-to-device upload)."""
    import torch
    import paper_2010_03166_b200 as gsg
    cfg = wl.CONFIGS[1]
    p = wl.parent_for(cfg).csr()
    ctx = gsg.Context(0)
    pg = gsg.ParentGraph(ctx, p.indptr, p.indices)
    batch = pg.sample(cfg.n, cfg.m, 99, count=1)
    ip, ix, nd = batch.tensors(0)
    sg = ctx.upload_device(ip, ix).normalize()
    ipn, ixn = ip.cpu().numpy(), ix.cpu().numpy()
    A = orc.normalize(ipn, ixn, orc.NORM_ROW_SELF)
    X = np.random.default_rng(0).standard_normal((sg.n, 56)).astype(np.float32)
    Y = torch.zeros((sg.n, 56), device="cuda")
    ctx.spmm(sg, torch.from_numpy(X).cuda(), Y)
    ref = orc.spmm(A, X)
    assert np.abs(Y.cpu().numpy() - ref).max() <= 1e-5 * np.abs(ref).max()


@pytest.mark.gpu
def test_gpu_sample_assign_and_gather():
    """A GPU sample refills an existing subgraph from device arrays (gsg_subgraph_assign with
    device pointers) bit for bit, and gsg_gather_rows builds X_s = X[V_s] and the labels
    (Alg. 1 line 5) exactly like a host gather of the same rows."""
    import torch
    import paper_2010_03166_b200 as gsg
    cfg = wl.CONFIGS[1]
    p = wl.parent_for(cfg).csr()
    ctx = gsg.Context(0)
    pg = gsg.ParentGraph(ctx, p.indptr, p.indices)
    batch = pg.sample(cfg.n, cfg.m, 123, count=2)
    g0 = wl.sample_subgraph(cfg)
    sg = ctx.upload(g0.indptr, g0.indices)
    rng = np.random.default_rng(5)
    Xp = rng.standard_normal((p.n, 50)).astype(np.float32)
    Lp = rng.integers(0, 255, size=(p.n, 7), dtype=np.uint8)
    Xpd = torch.zeros((p.n, 56), device="cuda")[:, :50]
    Xpd.copy_(torch.from_numpy(Xp))
    Lpd = torch.from_numpy(Lp).cuda()
    for k in range(2):
        info = batch.get(k)
        ip, ix, nd = (t.cpu().numpy() for t in batch.tensors(k))
        sg.assign(info["n"], info["nnz"], info["d_indptr"], info["d_indices"])
        sg.normalize()
        ref = orc.normalize(ip, ix, orc.NORM_ROW_SELF)
        dip, dix, _, _ = sg.download()
        assert np.array_equal(dip, ref.indptr) and np.array_equal(dix, ref.idx)
        Xs = torch.zeros((info["n"], 56), device="cuda")[:, :50]
        Ls = torch.zeros((info["n"], 7), dtype=torch.uint8, device="cuda")
        ctx.gather_rows(Xpd, info["d_nodes"], Xs, info["n"])
        ctx.gather_rows(Lpd, info["d_nodes"], Ls, info["n"])
        assert np.array_equal(Xs.cpu().numpy(), Xp[nd])
        assert np.array_equal(Ls.cpu().numpy(), Lp[nd])
    with pytest.raises(gsg.GsgError):  # device arrays cannot be validated on the host
        info = batch.get(0)
        sg.assign(info["n"], info["nnz"], info["d_indptr"], info["d_indices"], validate=True)


@pytest.mark.gpu
def test_gpu_sample_batches_reuse_buffers():
    """gsg_sample_free hands a batch's arrays back to its context and the next gsg_frontier_sample
    reuses them (gsg.h): a reused batch must equal a batch drawn in a fresh context, including
    a smaller second batch (fewer samples, different n) over the larger batch's stale contents; a
    batch freed after its context was destroyed frees its own arrays."""
    import paper_2010_03166_b200 as gsg
    p = parent(n=6000, deg=12.0, seed=7)
    ctx = gsg.Context(0)
    pg = gsg.ParentGraph(ctx, p.indptr, p.indices)
    first = pg.sample(900, 60, 11, count=5, clip=4)
    first.free()  # its arrays go to the context's pool
    second = pg.sample(700, 50, 22, count=3, clip=4)  # drawn into (some of) the reused arrays
    fresh_ctx = gsg.Context(0)
    fresh = gsg.ParentGraph(fresh_ctx, p.indptr, p.indices).sample(700, 50, 22, count=3, clip=4)
    for k in range(3):
        a, b = second.to_host(k), fresh.to_host(k)
        assert all(np.array_equal(x, y) for x, y in zip(a, b)), f"sample {k} differs after buffer reuse"
        v = orc.frontier_sample(p.indptr, p.indices, 700, 50, 4, sampler_seed(22, k))
        assert np.array_equal(a[2], v)
    fresh.free()
    fresh_ctx.close()
    third = pg.sample(900, 60, 33, count=2, clip=4)
    pg.free()
    ctx.close()  # destroys the context while `third` is alive
    third.free()  # frees its own arrays (no pool left)
    second.free()
