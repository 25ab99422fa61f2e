"""paper_2406_08334_b200 — B200-native ProTrain chunk hot path.

Layers:
  include/ptk.h + csrc/      C-ABI data plane for sm_100a (libptk.so): fused
                             chunk Adam, grad statistics, NCCL chunk AG/RS,
                             fused RS->Adam->AG over peer memory, host Adam
  include/memplan/ + csrc/planner/
                             clean-room drop-in of the reference planner API
                             (libmemplan.so + memplan CLI)
  chunks.py                  ZeRO-3 chunk buffers + step driver (host side)
  planner.py                 Python access to the planner (CLI / C-ABI)

Importing the package does not load CUDA; `from paper_2406_08334_b200 import
_native` loads libptk.so and raises if it is missing (no fallback).
"""
import os

PACKAGE_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PACKAGE_DIR)

__all__ = ["PACKAGE_DIR", "REPO_DIR"]
