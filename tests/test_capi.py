"""The C ABI library loads without a GPU and exports every entry point that
include/scmoe.h declares (no compute calls here)."""

import os
import re

import pytest

from paper_2404_05019_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "scmoe.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(scmoe_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = _declared()
    for n in ("scmoe_gate_topk", "scmoe_dispatch", "scmoe_grouped_gemm", "scmoe_expert_ffn",
              "scmoe_combine", "scmoe_last_error", "scmoe_version"):
        assert n in names


def test_library_exports_every_declared_symbol():
    so = _lib.load_library()
    for n in _declared():
        assert hasattr(so, n), n
    typed = {name for name, _, _ in _lib.SIGNATURES}
    assert typed == set(_declared())
    assert so.scmoe_version() == 2


def test_workspace_query_is_host_only():
    so = _lib.load_library()
    assert so.scmoe_gate_workspace_bytes(16384, 8, 2048) >= 256 + 2 * 256 * 8 * 4 + 32 * 3072


def test_argument_errors_do_not_touch_the_gpu():
    so = _lib.load_library()
    rc = so.scmoe_gate_topk(None, 1, 8, None, None, None, None, 0, 8, 4, 1, 1, None, None, None,
                            None, None, None, None, None, 0, None)
    assert rc == _lib.SCMOE_ERR_ARG
    assert b"n_tokens" in so.scmoe_last_error()
    rc = so.scmoe_combine(None, None, None, None, 7, None, None, None, None, 1, 1, 8, 1, 1,
                          None, None)
    assert rc == _lib.SCMOE_ERR_ARG


def test_sass_contains_tcgen05_and_tma():
    import shutil
    import subprocess
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not on PATH")
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UTCHMMA" in sass   # tcgen05.mma
    assert "UTMALDG" in sass   # TMA tensor load
    assert "LDTM" in sass      # tcgen05.ld


def test_host_queries_of_the_round_two_entries():
    """Workspace queries and argument checks of the entries added in round 2
    (two-matrix column sums, mean, aux loss, fill, the gate with sync words,
    the split fused combine) answer on the host."""
    so = _lib.load_library()
    one = so.scmoe_grouped_colsum_workspace_bytes(1, 18432, 384)
    two = so.scmoe_grouped_colsum2_workspace_bytes(1, 18432, 384, 1536)
    assert one > 0 and two > one
    assert so.scmoe_grouped_colsum2_workspace_bytes(1, 18432, 384, 0) == 0
    assert so.scmoe_mean_workspace_bytes() >= 4
    assert so.scmoe_gate_aux_loss(None, None, 0, 8, 1, None, None) == _lib.SCMOE_ERR_ARG
    assert so.scmoe_fill_div(None, 9, 8, None, 1.0, None) == _lib.SCMOE_ERR_ARG
    assert so.scmoe_mean(None, 1, 0, None, None, 0, None) == _lib.SCMOE_ERR_ARG
    rc = so.scmoe_gate_topk_ex(None, 1, 8, None, None, None, None, None, 0, 8, 4, 1, 1, None,
                               None, None, None, None, None, None, None, 0, None, None)
    assert rc == _lib.SCMOE_ERR_ARG and b"n_tokens" in so.scmoe_last_error()
    rc = so.scmoe_ffn2_combine(None, 0, None, None, None, None, None, None, None, 1, 1, None,
                               8, 8, 8, None)
    assert rc == _lib.SCMOE_ERR_ARG       # fp32: the fused combine runs on bf16


def test_gemm_sm_budget_nesting():
    """Nested SM budgets take the smaller and restore the outer on exit
    (the concurrent backward nests a side budget in the main one)."""
    from paper_2404_05019_b200 import kernels as K
    assert K._SM_BUDGET[0] == 0
    with K.gemm_sm_budget(74):
        assert K._SM_BUDGET[0] == 74
        with K.gemm_sm_budget(96):
            assert K._SM_BUDGET[0] == 74
        with K.gemm_sm_budget(16):
            assert K._SM_BUDGET[0] == 16
        assert K._SM_BUDGET[0] == 74
        with K.gemm_sm_budget(0):
            assert K._SM_BUDGET[0] == 74
    assert K._SM_BUDGET[0] == 0
