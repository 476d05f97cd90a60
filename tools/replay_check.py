"""Set-up check of the matrix-free phase B: BCT_CHECK_REPLAY=1 makes the
library replay every recorded forward segment and compare it with the stored
entries (prints mismatching segments per panel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BCT_CHECK_REPLAY"] = "1"
from paper_1709_00953_b200 import CONFIGS, DeviceBlockSystem  # noqa

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
DeviceBlockSystem.parallel_beam(cfg.spec, dtype=sys.argv[2] if len(sys.argv) > 2 else cfg.dtype)
