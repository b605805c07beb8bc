"""Seeded synthetic inputs shared by the CPU oracle and the CUDA path (data only)."""
from .spec import *  # noqa: F401,F403
from .spec import agg_words
from .templates import paper11, paper11_variants, toy2, w1, w2, w3, w4, w6, w7, w8, w9, w10, w11
from .configs import CONFIGS, get_config

__all__ = ["paper11", "paper11_variants", "toy2", "w1", "w2", "w3", "w4", "w6", "w7", "w8", "w9", "w10", "w11", "CONFIGS", "get_config", "agg_words"]
