"""Learner-side roles and cross-role synchronisation on the device
(mirror of the learner sections of R:runtime/__init__.py:17-33)."""

from ..errors import PipelineStall
from .learners import (AppoLearner, PpoLearner, SacLearner, build_ac_params, run_appo,
                       run_ppo_sync)
from .sac_pipeline import SacPipeline, stream
from .sync import (ErrorBox, HostAcParams, HostParams, RolloutRing, WeightSlot, fetch_weights,
                   publish_weights)

__all__ = ["AppoLearner", "ErrorBox", "HostAcParams", "HostParams", "PipelineStall",
           "PpoLearner", "RolloutRing", "SacLearner", "SacPipeline", "WeightSlot", "build_ac_params",
           "fetch_weights", "publish_weights", "run_appo", "run_ppo_sync", "stream"]
