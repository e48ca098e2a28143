"""Run a script against the experiments build of the library (A/B knobs read
from the environment): python tools/with_ab_lib.py SCRIPT [ARGS...].
Tools only -- the product path never loads build/ab/."""
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_17001_b200._lib as _L  # noqa: E402

_L.LIB_PATH = os.environ.get("ICNNM_AB_LIB_FILE") or os.path.join(ROOT, "build", "ab", "libicnnm_b200_ab.so")
script = sys.argv[1]
sys.argv = sys.argv[1:]
runpy.run_path(script, run_name="__main__")
