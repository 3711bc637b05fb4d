"""Developer timing probe (not a test, not the bench): V1309 max-level-13 inputs
from the oracle's moments, all levels in one fused compute, CUDA-event timing.
Usage: python tests/perf_probe.py [max_level] [theta]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1908_03121_b200 as P  # noqa: E402
from gpu_util import api_inputs  # noqa: E402


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 13
    theta = float(sys.argv[2]) if len(sys.argv) > 2 else 0.34
    t0 = time.time()
    tr = synth.config_v1309(L)
    mom = oracle.moments(tr)
    print("tree", tr.summary()["subgrids"], "subgrids", tr.summary()["refined"], "refined",
          f"build {time.time() - t0:.1f}s", flush=True)
    f = P.OctoFMM(theta)
    for lv in tr.levels[1:]:
        mono, com, mm = (torch.from_numpy(a).cuda() for a in api_inputs(tr, mom, lv.level))
        f.load_level(lv.level, lv.h, tr.origin, lv.ijk, lv.refined, lv.neighbors, None, mono, com, mm)
        torch.cuda.synchronize()
    cnt = f.interaction_counts()
    print("interactions p2p/m2l/mixed", cnt.tolist(), flush=True)
    st = torch.cuda.current_stream()
    for _ in range(3):
        f.compute_interactions()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        f.compute_interactions()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    print(f"compute_interactions(ALL): median {ms:.3f} ms, min {min(ts):.3f} ms; "
          f"{cnt.sum() / ms / 1e6:.2f} G interactions/s "
          f"(m2l+mixed {(cnt[1] + cnt[2]) / 1e6:.1f} M, p2p {cnt[0] / 1e6:.1f} M)")
    # per-class: separate handles with only refined / only leaf work are not
    # exposed; time per level instead
    for lv in tr.levels[1:]:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        f.compute_interactions(lv.level)
        b.record(st)
        b.synchronize()
        c = f.interaction_counts(lv.level)
        print(f"  level {lv.level:2d}: nodes {lv.n_nodes:5d} refined {lv.n_refined:5d} "
              f"{a.elapsed_time(b):8.3f} ms  p2p {c[0] / 1e6:8.1f}M m2l {c[1] / 1e6:7.1f}M mix {c[2] / 1e6:6.1f}M")


if __name__ == "__main__":
    main()
