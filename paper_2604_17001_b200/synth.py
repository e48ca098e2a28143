"""Re-export of the BASELINE input generator (test / bench infrastructure).

The generator lives outside the product in ``synthgen`` (its own host-only
library), so the product library never carries it and the reference arm of
bench.py never loads the product; tests keep importing it from here.
"""
import os as _os
import sys as _sys

_ROOT = _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))
if _ROOT not in _sys.path:
    _sys.path.insert(0, _ROOT)

from synthgen import *  # noqa: E402,F401,F403
from synthgen import (MASK_IID, MASK_EXACT, MASK_T_FRAMES, MASK_T_PREFIX,  # noqa: E402,F401
                      MASK_IID_BOXES, Rng, Workload, WORKLOADS, psnr, reference_bernoulli_mask,
                      scaled, synth_mask, synth_video)
