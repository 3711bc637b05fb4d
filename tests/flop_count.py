"""Per-interaction FP64 flop counts of the shipped kernels, derived from the
SASS of libocto_fmm.so (C10 and §5).

Convention: DFMA = 2 flops, DMUL / DADD = 1, MUFU.RSQ64H (the FP64 rsqrt seed)
= 1; integer, address and shared-memory instructions are not flops.  The count
is the op count of the formula the kernels actually evaluate (the detraced
order-3 M2L with the AM correction; P2P with the precomputed K(d) geometry),
so it drifts with kernel edits -- tests/test_flop_count.py pins bench.py's
constants to this script's output.

How: every innermost FP64 loop of a kernel is located in the SASS (a
backward branch closing a range with FP64 work that contains no other such
range).  Each M2L /
mixed pair issues exactly one MUFU.RSQ64H, so flops per pair = the loop's
flops / its MUFU count (every innermost pair loop must agree).  The P2P row
loop holds the specialised row bodies (x half-width XR = 0, 1, 2; each may be
compiled in several copies), 8 child parities x 4 targets x (2 XR + 1) parent
offsets each, and nothing but DFMAs: 4 per interaction.

Usage: python tests/flop_count.py [path/to/libocto_fmm.so]   (prints JSON)
"""
from __future__ import annotations

import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1908_03121_b200", "libocto_fmm.so")

# the kernels the bench launches (default configuration: AM correction on,
# parent reach 2 (theta >= 1/3), M2L with 2 pairs per far-loop iteration)
KERNELS = {
    "m2l": r"m2l_dense_kernelILb1ELi2ELi2E",
    "mixed": r"m2l_mixed_kernelILb1ELi2ELb0E",
    "p2p": r"p2p8_kernelILi2E",
}


def sass(lib=LIB):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs = {}
    for chunk in re.split(r"\n\s*Function : ", out)[1:]:
        name = chunk.split("\n", 1)[0].strip()
        ins = []
        for line in chunk.split("\n"):
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
            if m:
                ins.append((int(m.group(1), 16), m.group(2)))
        funcs[name] = ins
    return funcs


def _count(body):
    def c(op):
        return sum(1 for t in body if re.search(r"(^|\s)" + op + r"(\.\S+)?\s", t))
    return {"DFMA": c("DFMA"), "DMUL": c("DMUL"), "DADD": c("DADD"),
            "MUFU": sum(1 for t in body if "MUFU.RSQ64H" in t)}


def innermost_loops(ins):
    addr = {a: i for i, (a, _) in enumerate(ins)}
    loops = []
    for i, (a, t) in enumerate(ins):
        m = re.search(r"\bBRA\b.*?(0x[0-9a-f]+)", t)
        if m:
            tg = int(m.group(1), 16)
            if tg <= a and tg in addr:
                loops.append((addr[tg], i))
    cnt = {r: _count([t for _, t in ins[r[0]:r[1] + 1]]) for r in loops}
    fp = [r for r in loops if cnt[r]["DFMA"] + cnt[r]["DMUL"] > 10]
    # innermost FP loops: no other FP loop nested inside (an integer-only
    # inner loop, e.g. the mixed kernel's advance to the next slot, is allowed)
    inner = [(s, e) for (s, e) in fp if not any((s2, e2) != (s, e) and s <= s2 and e2 <= e for s2, e2 in fp)]
    return [cnt[r] for r in inner]


def flops(n):
    return 2 * n["DFMA"] + n["DMUL"] + n["DADD"] + n["MUFU"]


def derive(lib=LIB):
    funcs = sass(lib)
    res = {}
    for key, pat in KERNELS.items():
        names = [f for f in funcs if re.search(pat, f)]
        assert len(names) >= 1, (key, names)
        # several instantiations (e.g. M2L whole / half stages) share the pair loop
        assert all(innermost_loops(funcs[n]) == innermost_loops(funcs[names[0]]) for n in names), (key, names)
        loops = innermost_loops(funcs[names[0]])
        if key == "p2p":
            # only DFMAs (4 per target-partner pair, K(d) precomputed); the row
            # loop holds the XR = 0, 1, 2 bodies (each possibly in several
            # specialised copies): per body 2 partner parities qy x 8 targets x
            # (4 XR + 2) partner children (p2p8_kernel: both qx planes, parent
            # offsets -XR..XR), 4 DFMA each
            assert len(loops) == 1, loops
            n = loops[0]
            inter = sum(2 * 8 * (4 * xr + 2) for xr in (0, 1, 2))
            assert n["DMUL"] == 0 and n["DADD"] == 0 and n["MUFU"] == 0, n
            assert n["DFMA"] % (4 * inter) == 0, (n, inter)
            res[key] = {"flop": 2 * 4, "sass_loop": n, "interactions_per_body_set": inter,
                        "body_copies": n["DFMA"] // (4 * inter)}
        else:
            # pair loops: one MUFU.RSQ64H per pair (FP64 loops without one, e.g. a
            # rotated loop tail or a fix-up block, are not pair loops)
            per = []
            for n in loops:
                if n["MUFU"] == 0:
                    continue
                per.append(flops(n) / n["MUFU"])
            assert per and max(per) == min(per), (key, loops)
            assert per[0] == int(per[0]), (key, per)
            res[key] = {"flop": int(per[0]), "sass_loops": loops}
    return res


if __name__ == "__main__":
    print(json.dumps(derive(sys.argv[1] if len(sys.argv) > 1 else LIB), indent=1))
