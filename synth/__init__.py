"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic: only counter-based random bits (``rng``) and
the placement of tokens into blocks (``workload``).  See DESIGN.md "Input recipe".
"""
from .workload import (CONFIGS, Workload, make_config, materialize_numpy, materialize_torch,  # noqa: F401
                       shard, subset, tables_torch)
