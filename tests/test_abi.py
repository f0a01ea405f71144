"""C-ABI boundary checks that need no GPU: libgsg.so loads, exports every symbol include/gsg.h
declares, and refuses to run (loudly) where there is no sm_100 device."""
import ctypes
import subprocess

import pytest

import paper_2010_03166_b200 as gsg
from conftest import cuda_available


def test_header_declares_the_boundary():
    names = set(gsg.exported_symbols())
    # upload/normalize, layer_forward, layer_backward, allreduce_grads
    for required in ["gsg_subgraph_upload", "gsg_subgraph_normalize", "gsg_layer_forward", "gsg_layer_backward",
                     "gsg_allreduce_grads", "gsg_spmm", "gsg_gemm", "gsg_head", "gsg_ctx_create", "gsg_last_error"]:
        assert required in names, required


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", gsg.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for name in gsg.exported_symbols():
        assert name in exported, f"{name} declared in gsg.h but not exported"
        assert hasattr(gsg, name), f"{name} has no Python binding"
    # nothing else leaks out of the library (hidden visibility)
    leaked = [s for s in exported if s.startswith("gsg") and s not in set(gsg.exported_symbols())]
    assert not leaked, leaked


def test_library_contains_tcgen05_and_tma():
    """The GEMM is a tcgen05 kernel (UTC*MMA, LDTM) fed by TMA (UTMALDG): B200_PROFILING.md table."""
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", gsg.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCQMMA" in sass
    assert "UTMALDG" in sass and "LDTM" in sass
    assert "HMMA" not in sass.replace("UTCHMMA", "")  # no legacy mma.sync path


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU failure path")
def test_context_fails_loudly_without_gpu():
    with pytest.raises(gsg.GsgError):
        gsg.Context(0)
    assert gsg.last_error() != ""


def test_null_context_is_rejected():
    assert gsg.gsg_ctx_sync(None) == gsg.GSG_EINVAL
    assert "NULL context" in gsg.last_error()
    assert gsg.gsg_nccl_unique_id(None) == gsg.GSG_EINVAL
