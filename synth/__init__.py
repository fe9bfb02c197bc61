"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the A^2ATS method: it only draws random
numbers (torch.Generator, any device) and lays them out in the shapes the
boundary takes.  Values the method computes (rotations, scores, codes from
encoding, selections, attention) never appear here.
"""
from .configs import CONFIGS, Config, budget_k  # noqa: F401
from .generators import make_inputs, make_codebook, make_h, make_query  # noqa: F401
