"""pi0b: a B200-native (sm_100a) pi0 inference engine."""
from .config import ModelConfig, default_config, mid_config, tiny_config  # noqa: F401
