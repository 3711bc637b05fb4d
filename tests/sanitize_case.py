"""Small end-to-end case for compute-sanitizer runs (not a test): every
kernel of the library on configs[2] levels 0-3 (root, M2L, mixed, P2P, prep,
P2M/M2M, L2L, field, compact getter)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1908_03121_b200 as P  # noqa: E402
from paper_1908_03121_b200.levels import upward, load_tree  # noqa: E402

tr = synth.config_c3()
f = P.OctoFMM(0.34, timing=True)
data = upward(f, tr)
load_tree(f, tr, data)
f.compute_interactions()
f.compute_interactions(2)
f.propagate()
for lv in tr.levels:
    phi = torch.zeros((lv.n_nodes, 512), dtype=torch.float64, device="cuda")
    g = torch.zeros((3, lv.n_nodes, 512), dtype=torch.float64, device="cuda")
    f.get_field(lv.level, phi, g)
    nr, nf = f.compact_sizes(lv.level)
    R = np.zeros((23, nr, 512))
    F = np.zeros((7, nf, 512))
    f.get_expansions_compact(lv.level, R, F)
f.sync()
print("sanitize case ok", f.kernel_times()[1], f.launch_count())
