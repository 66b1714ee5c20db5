"""B200-native ScMoE layer (arXiv 2404.05019): hand-written sm_100a kernels
behind the reference's module API.  See DESIGN.md."""

from .layers import (CapacityConfig, ConfigError, GateDecision, MoEReplay, RoutedExperts,
                     ScMoELayer, SharedExpert, Top1Gate, Top2MoELayer)
from .kernels import expert_quota
from .block import Attention, ScMoEBlockPair
from . import sched, timeline, ep

__all__ = ["CapacityConfig", "ConfigError", "GateDecision", "MoEReplay", "RoutedExperts",
           "ScMoELayer", "SharedExpert", "Top1Gate", "Top2MoELayer", "expert_quota",
           "Attention", "ScMoEBlockPair", "sched", "timeline", "ep"]
from .block import ScMoEBlock, ScMoEModel
from .layers import DGMoELayer
__all__ += ["ScMoEBlock", "ScMoEModel", "DGMoELayer"]
