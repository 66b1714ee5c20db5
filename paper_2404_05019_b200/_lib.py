"""ctypes binding of libscmoe.so (the C ABI declared in include/scmoe.h).

This is the reference-facing boundary: every hot-path call of the package
goes through these functions.  There is no CPU fallback — if the library or
an sm_100 device is missing, `lib()` raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SCMOE_LIB overrides the library path (A/B of two builds in one session)
LIB_PATH = os.environ.get("SCMOE_LIB") or os.path.join(_HERE, "libscmoe.so")

SCMOE_OK, SCMOE_ERR_ARG, SCMOE_ERR_CUDA, SCMOE_ERR_UNSUPPORTED = 0, 1, 2, 3
SCMOE_F32, SCMOE_BF16 = 0, 1
COMBINE_MODES = {"direct_add": 0, "cg1": 1, "cg2": 2}
EPI_BIAS, EPI_BIAS_GELU, EPI_GELU_BWD, EPI_MUL_AUX = 0, 1, 2, 3
W_NK, W_KN = 0, 1
MAX_EXPERTS, MAX_K = 64, 8

_vp, _i, _ll, _sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_size_t

# (name, restype, argtypes) — keep in sync with include/scmoe.h
SIGNATURES = [
    ("scmoe_version", _i, []),
    ("scmoe_last_error", ctypes.c_char_p, []),
    ("scmoe_device_check", _i, [_i]),
    ("scmoe_gate_workspace_bytes", _sz, [_i, _i, _i]),
    ("scmoe_gate_topk", _i, [_vp, _i, _ll, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i,
                             _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    ("scmoe_gate_split_bytes", _sz, [_i, _i]),
    ("scmoe_gate_split_weights", _i, [_vp, _i, _i, _vp, _vp]),
    ("scmoe_gate_topk_presplit", _i, [_vp, _i, _ll, _vp, _vp, _vp, _i, _i, _i, _i, _i,
                                      _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    ("scmoe_gate_topk_ex", _i, [_vp, _i, _ll, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i,
                                _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _vp]),
    ("scmoe_dispatch", _i, [_vp, _i, _ll, _i, _i, _i, _vp, _vp, _i, _vp, _vp]),
    ("scmoe_grouped_gemm", _i, [_vp, _i, _vp, _vp, _vp, _vp, _i, _i, _i, _vp, _i, _i, _i, _i,
                                _vp]),
    ("scmoe_set_gemm_mode", _i, [_i]),
    ("scmoe_set_gemm_tile_n", _i, [_i]),
    ("scmoe_set_gemm_flags", _i, [_i]),
    ("scmoe_set_gemm_epilogue_warps", _i, [_i]),
    ("scmoe_set_gemm_sm_budget", _i, [_i]),
    ("scmoe_gather_rows", _i, [_vp, _sz, _vp, _vp, _i, _vp, _vp]),
    ("scmoe_copy_rows", _i, [_vp, _sz, _vp, _i, _vp, _vp]),
    ("scmoe_sgd_update", _i, [_vp, _vp, _vp, _vp, _i, ctypes.c_float, _vp]),
    ("scmoe_grouped_gemm_ex", _i, [_vp, _i, _vp, _i, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _vp,
                                   _i, _i, _i, _i, _i, _vp]),
    ("scmoe_grouped_wgrad_workspace_bytes", _sz, [_i, _i, _i, _i]),
    ("scmoe_grouped_wgrad", _i, [_vp, _vp, _i, _vp, _vp, _sz, _i, _i, _i, _vp, _i, _i, _i, _i,
                                 _vp]),
    ("scmoe_grouped_wgrad_ex", _i, [_vp, _vp, _i, _vp, _i, _vp, _sz, _i, _i, _i, _vp, _i, _i, _i,
                                    _i, _vp]),
    ("scmoe_zero_tails", _i, [_vp, _i, _i, _i, _i, _vp, _i, _i, _vp]),
    ("scmoe_grouped_colsum_workspace_bytes", _sz, [_i, _i, _i]),
    ("scmoe_grouped_colsum", _i, [_vp, _i, _i, _i, _i, _vp, _i, _vp, _vp, _sz, _vp]),
    ("scmoe_gate_aux_loss", _i, [_vp, _vp, _i, _i, _i, _vp, _vp]),
    ("scmoe_fill_div", _i, [_vp, _i, ctypes.c_longlong, _vp, ctypes.c_float, _vp]),
    ("scmoe_mean_workspace_bytes", _sz, []),
    ("scmoe_mean", _i, [_vp, _i, ctypes.c_longlong, _vp, _vp, _sz, _vp]),
    ("scmoe_grouped_colsum2_workspace_bytes", _sz, [_i, _i, _i, _i]),
    ("scmoe_grouped_colsum2", _i, [_vp, _vp, _i, _i, _i, _i, _i, _vp, _i, _vp, _vp, _vp, _sz, _vp]),
    ("scmoe_dispatch_scaled", _i, [_vp, _i, _ll, _i, _i, _i, _vp, _vp, _i, _vp, _vp, _vp]),
    ("scmoe_expert_ffn", _i, [_vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _vp, _i,
                              _i, _i, _vp]),
    ("scmoe_combine", _i, [_vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i,
                           _vp, _vp]),
    ("scmoe_ep_dispatch_p2p", _i, [_vp, _i, _ll, _i, _i, _i, _vp, _vp, _vp, _i, _i, _i, _i,
                                   _vp, _vp, _vp, _vp, _i, _vp]),
    ("scmoe_ep_wait", _i, [_vp, _i, _i, _vp, _vp]),
    ("scmoe_ep_signal", _i, [_vp, _i, _i, _i, _vp, _vp]),
    ("scmoe_ep_combine_p2p", _i, [_vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i,
                                  _i, _i, _i, _vp, _vp]),
    ("scmoe_shared_ffn_combine", _i, [_vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                      _i, _i, _vp, _vp, _i, _i, _i, _vp]),
    ("scmoe_ffn2_combine", _i, [_vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp, _i, _i,
                                _i, _vp]),
    ("scmoe_pack_heads", _i, [_vp, _vp, _i, _i, _i, _i, _i, _i, _vp, _vp]),
    ("scmoe_expert_ffn_to_peers", _i, [_vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _vp,
                                       _i, _i, _i, _vp]),
    ("scmoe_ep_return_p2p", _i, [_vp, _i, _vp, _i, _i, _i, _i, _i, _vp, _vp, _vp, _i, _vp]),
    ("scmoe_window_attention_supported", _i, [_i, _i]),
    ("scmoe_window_attention_fwd", _i, [_vp, _i, _i, _i, _i, ctypes.c_float, _i, _vp, _vp, _vp]),
    ("scmoe_window_attention_bwd", _i, [_vp, _vp, _vp, _vp, _i, _i, _i, _i, ctypes.c_float, _i,
                                        _vp, _vp]),
    ("scmoe_gelu_fwd", _i, [_vp, _vp, _i, _i, _i, _vp, _i, _vp]),
    ("scmoe_gelu_fwd_grad", _i, [_vp, _vp, _vp, _i, _i, _i, _vp, _i, _vp]),
    ("scmoe_gelu_bwd_workspace_bytes", _sz, [_i, _i, _i]),
    ("scmoe_gelu_bwd", _i, [_vp, _vp, _vp, _vp, _i, _i, _i, _vp, _i, _vp, _sz, _vp]),
    ("scmoe_gate_backward_workspace_bytes", _sz, [_i, _i, _i, _i]),
    ("scmoe_gate_backward", _i, [_vp, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                 _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
]

_lib = None
_lock = threading.Lock()
_checked_devices = set()


class ScMoEError(RuntimeError):
    """CUDA-side failure inside libscmoe."""


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load and type the library without touching a GPU (used by CPU tests)."""
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " or `make -C paper_2404_05019_b200/csrc`")
    so = ctypes.CDLL(path)
    for name, res, args in SIGNATURES:
        # an A/B against an older build (SCMOE_LIB) may lack newer entries
        fn = getattr(so, name, None) if os.environ.get("SCMOE_LIB") else getattr(so, name)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    return so


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                _lib = load_library()
    return _lib


def check(rc: int) -> None:
    if rc == SCMOE_OK:
        return
    msg = lib().scmoe_last_error().decode(errors="replace")
    if rc == SCMOE_ERR_ARG:
        raise ValueError(msg)
    raise ScMoEError(f"libscmoe error {rc}: {msg}")


def ensure_device(t: torch.Tensor) -> None:
    """Fail loudly unless `t` lives on an sm_100 GPU."""
    if not t.is_cuda:
        raise RuntimeError("paper_2404_05019_b200 runs on CUDA tensors only (no CPU fallback); "
                           f"got a tensor on {t.device}")
    dev = t.device.index if t.device.index is not None else torch.cuda.current_device()
    if dev not in _checked_devices:
        check(lib().scmoe_device_check(dev))
        _checked_devices.add(dev)


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def dtype_code(dtype: torch.dtype) -> int:
    if dtype == torch.bfloat16:
        return SCMOE_BF16
    if dtype == torch.float32:
        return SCMOE_F32
    raise ValueError(f"unsupported dtype {dtype}; use torch.bfloat16 or torch.float32")
