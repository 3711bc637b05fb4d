"""Developer probe (not a test): CUDA-event timeline of the pipelined e2e loop
(bench.py's e2e leg): per step, when ingest, kernels and result copies end."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1908_03121_b200 as P  # noqa: E402
from paper_1908_03121_b200.levels import upward  # noqa: E402

NH = int(os.environ.get("NH", "3"))
tree = synth.config_v1309(13)
lvls = list(tree.levels)
hs = [P.OctoFMM(0.34) for _ in range(NH)]
data = upward(hs[0], tree)
torch.cuda.synchronize()
host = {lv.level: {k: (v.cpu().pin_memory() if v is not None else None) for k, v in data[lv.level].items()} for lv in lvls}
ss = [torch.cuda.Stream() for _ in range(NH)]
outs = []
for i in range(NH):
    o = {}
    for lv in lvls:
        hs[i].load_level(lv.level, lv.h, tree.origin, lv.ijk, lv.refined, lv.neighbors, None,
                         host[lv.level]["mono"], host[lv.level]["com"], host[lv.level]["mom"], stream=ss[i])
        nr, nf = hs[i].compact_sizes(lv.level)
        o[lv.level] = (torch.empty((23, nr, 512), dtype=torch.float64).pin_memory(),
                       torch.empty((7, nf, 512), dtype=torch.float64).pin_memory())
    outs.append(o)
chain = {}
EV = []


def phase(s, name, k):
    if name in chain:
        s.wait_event(chain[name])
    e = torch.cuda.Event(enable_timing=True)
    chain[name] = e
    EV.append((k, name, e))
    return e


def step(k):
    i = k % NH
    f, s, o = hs[i], ss[i], outs[i]
    e = phase(s, "h2d", k)
    for lv in lvls:
        d = host[lv.level]
        f.load_level(lv.level, lv.h, tree.origin, lv.ijk, lv.refined, lv.neighbors, None, d["mono"], d["com"],
                     d["mom"], stream=s)
    e.record(s)
    e = phase(s, "compute", k)
    f.compute_interactions(stream=s)
    e.record(s)
    e = phase(s, "d2h", k)
    for lv in lvls:
        f.get_expansions_compact(lv.level, o[lv.level][0], o[lv.level][1], stream=s, non_blocking=True)
    e.record(s)


for k in range(NH):
    step(k)
torch.cuda.synchronize()
EV.clear()
base = torch.cuda.Event(enable_timing=True)
base.record()
for s in ss:
    s.wait_stream(torch.cuda.current_stream())
n = 12
for k in range(n):
    step(k)
torch.cuda.synchronize()
for k, name, e in EV:
    print(f"step {k:2d} {name:8s} ends {base.elapsed_time(e):8.2f} ms")
print(f"{NH} handles: {base.elapsed_time(EV[-1][2]) / n:.2f} ms/step")
