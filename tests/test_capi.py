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
