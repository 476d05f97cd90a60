"""Profiling helper: per-panel layout sizes (BCT_VERBOSE=1 prints them)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BCT_VERBOSE"] = "1"
from paper_1709_00953_b200 import CONFIGS, DeviceBlockSystem  # noqa

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
DeviceBlockSystem.parallel_beam(cfg.spec, dtype=cfg.dtype)
