"""Drop-in shim for the reference model: route `arch.moe_shared` and
`arch.moe_standard` (scmoelab/arch.py:489-504) through the B200 kernels so
that `arch.model_forward` / `arch.forward` run unchanged with the MoE layers
on the GPU.

    from paper_2404_05019_b200 import compat
    compat.install()          # patches scmoelab.arch in place
    out, trace = arch.forward(cfg, params, tokens)
    compat.uninstall()

Only value-mode calls (ndarray parameter leaves) are supported; tape.Tensor
leaves (gradient checking) raise — there is no CPU fallback.  Noise draws use
the caller's `rng` exactly as the reference does (rng.normal((T, N)),
arch.py:411-413), so replays stay bit-identical.
"""

from __future__ import annotations

import numpy as np
import torch

_saved = {}


def _is_tape(v) -> bool:
    return type(v).__name__ == "Tensor" and hasattr(v, "parents")


def _reference_decision(gating_mod, dec, eps):
    d = dec.to_numpy()
    return gating_mod.GateDecision(logits=d["logits"], indices=d["indices"], weights=d["weights"],
                                   dropped=d["dropped"], eps=eps)


def install(arch_module=None, dtype: torch.dtype = torch.float32, device: str = "cuda",
            gating_module=None):
    """Rebind arch.moe_shared / arch.moe_standard to GPU implementations.

    `arch_module` / `gating_module` default to the reference's scmoelab.arch /
    scmoelab.gating; any objects with the same attributes work (the tests use
    the oracle's)."""
    if arch_module is None:
        from scmoelab import arch as arch_module  # the reference package
    if gating_module is None:
        from scmoelab import gating as gating_mod
    else:
        gating_mod = gating_module
    from .layers import MoEReplay, ScMoELayer, Top2MoELayer

    if id(arch_module) in _saved:
        return
    _saved[id(arch_module)] = (arch_module.moe_shared, arch_module.moe_standard)

    def _prepare(x, layer, rng, replay):
        if _is_tape(x) or _is_tape(layer.gate.w_gate):
            raise NotImplementedError("GPU ScMoE layer runs value-mode forwards only")
        t, n = np.asarray(x).shape[0], np.asarray(layer.gate.w_gate).shape[1]
        eps = replay.eps if replay is not None else None
        if layer.gate.noise_enabled and eps is None:
            if rng is None:
                raise ValueError("noise enabled but neither rng nor recorded draws given")
            eps = rng.normal((t, n))
        pin = None
        if replay is not None and replay.indices is not None:
            pin = MoEReplay(indices=replay.indices, dropped=replay.dropped)
        return eps, pin

    def _t(a):
        return torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float64)),
                               device=device).to(dtype).contiguous()

    def moe_shared(x, layer, capacity, k, rng=None, replay=None, routed_src=None):
        eps, pin = _prepare(x, layer, rng, replay)
        m = ScMoELayer.from_reference(layer, capacity, dtype=dtype, device=device)
        with torch.no_grad():
            out, dec, aux = m(_t(x), None if routed_src is None else _t(routed_src),
                              eps=None if eps is None else _t(eps).float(), replay=pin)
        return (out.double().cpu().numpy(), _reference_decision(gating_mod, dec, eps),
                np.array([[float(aux)]]))

    def moe_standard(x, layer, capacity, k, rng=None, replay=None):
        eps, pin = _prepare(x, layer, rng, replay)
        m = Top2MoELayer.from_reference(layer, capacity, k=k, dtype=dtype, device=device)
        with torch.no_grad():
            out, dec, aux = m(_t(x), eps=None if eps is None else _t(eps).float(), replay=pin)
        return (out.double().cpu().numpy(), _reference_decision(gating_mod, dec, eps),
                np.array([[float(aux)]]))

    arch_module.moe_shared = moe_shared
    arch_module.moe_standard = moe_standard


def uninstall(arch_module=None):
    """Restore the reference implementations."""
    if arch_module is None:
        from scmoelab import arch as arch_module
    if id(arch_module) in _saved:
        arch_module.moe_shared, arch_module.moe_standard = _saved.pop(id(arch_module))
