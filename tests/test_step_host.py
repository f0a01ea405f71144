"""Host-side logic of the training step (no GPU): the §7.1 chain-order rule and the
work counts bench.py divides by (2 nnz' f edge-features per layer for a2 + a7, f
the width the aggregation runs at; 6 n f_in f_out GEMM flops per layer)."""
import pytest

pytest.importorskip("torch")
import paper_2010_03166_b200.step as step_mod  # noqa: E402  (binding import needs libgsg.so, not a GPU)


def fake_step(dims, head="none", classes=0):
    s = object.__new__(step_mod.GCNStep)
    s.dims, s.L, s.head, s.C = list(dims), len(dims) - 1, head, classes
    s.order = [step_mod.chain_order(dims[l], dims[l + 1]) for l in range(s.L)]
    return s


def test_chain_order_rule():
    # (ÂX)W costs δn²·f_in + n f_in f_out MACs, Â(XW) δn²·f_out + n f_in f_out: order 2 iff f_in > f_out
    assert step_mod.chain_order(602, 512) == 2
    assert step_mod.chain_order(200, 1024) == 1
    assert step_mod.chain_order(1024, 1024) == 1   # tie keeps the north star's order
    assert step_mod.chain_order(50, 128) == 1


def test_work_counts_config5_and_config2():
    s5 = fake_step([200, 1024, 1024, 1024], "sigmoid", 107)
    nh = 2_352_360
    assert s5.work_edge_features(nh) == 2 * nh * (200 + 1024 + 1024)
    # training mode: layer 1's a7 (width f_0 under order 1) is not run
    assert s5.work_edge_features(nh, input_grad=False) == 2 * nh * (200 + 1024 + 1024) - nh * 200
    n = 20_000
    assert s5.gemm_flops(n) == 6 * n * (200 * 1024 + 2 * 1024 * 1024) + 6 * n * 1024 * 107
    s2 = fake_step([602, 512, 512], "softmax", 41)
    assert s2.order == [2, 1]
    # order 2 on layer 1: both aggregations run at f_out = 512; its G = Âᵀ dZ still feeds dW
    assert s2.work_edge_features(100) == 2 * 100 * (512 + 512)
    assert s2.work_edge_features(100, input_grad=False) == s2.work_edge_features(100)


def test_ld_for_alignment():
    assert step_mod.ld_for(200) == 200 and step_mod.ld_for(201) == 208 and step_mod.ld_for(5, 4) == 8
