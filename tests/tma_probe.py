"""Developer probe (not a test): one configs[2] compute with the TMA-staged
mixed kernel under a short timeout, checked against the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle  # noqa: E402
import synth  # noqa: E402
from gpu_util import get, load, parity  # noqa: E402
import paper_1908_03121_b200 as P  # noqa: E402

tr = synth.config_c3()
mom = oracle.moments(tr)
for level in (2, 3):
    f = P.OctoFMM(0.34)
    load(f, tr, mom, level)
    f.compute_interactions(level)
    L, Lc = get(f, tr, level)
    oL, oLc, oab = oracle.same_level(tr, mom, level, 0.34)
    print("level", level, "parity", parity(L.reshape(20, -1).T, Lc.reshape(3, -1).T, oL, oLc, oab), flush=True)
    f.close()
