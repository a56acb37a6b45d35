"""B200-native AGILE async page-I/O hot path (arxiv 2504.19365), drop-in for ``agile_sim``'s
import surface (reference ``__init__.py:5-10``): AgileSystem, ExperimentConfig, SystemConfig,
TraceRecorder.  The compute path is the native library ``libagile_b200.so`` (sm_100a); there is
no CPU fallback."""

from .config import ExperimentConfig, SystemConfig
from .system import AgileSystem
from .trace import TraceRecorder

__all__ = ["AgileSystem", "ExperimentConfig", "SystemConfig", "TraceRecorder"]
