"""Tuning harness (not a test): build library variants with extra nvcc
defines here (cross-compile), then time each on the GPU box with the bench's
own step (configs[3], kernel times from the library's CUDA events).

  python tests/perf_variants.py build NAME=-DFOO=1,-DBAR=2 NAME2=...   # here
  python tests/perf_variants.py run [--steps K] [--env NAME:K=V,...]    # on the GPU box

Variants live in paper_1908_03121_b200/variants/ (git-ignored *.so, they
travel to the box with the snapshot); `run` prints one JSON line per variant.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VDIR = os.path.join(ROOT, "paper_1908_03121_b200", "variants")


def build(specs):
    sys.path.insert(0, ROOT)
    from paper_1908_03121_b200 import build as b
    os.makedirs(VDIR, exist_ok=True)
    for spec in specs:
        name, _, flags = spec.partition("=")
        out = os.path.join(VDIR, f"lib_{name}.so")
        b.build(out=out, extra=[f for f in flags.split(",") if f])
        print("built", out, flush=True)


def run(argv):
    steps = "20"
    envs = {}
    names = None
    i = 0
    while i < len(argv):
        if argv[i] == "--steps":
            steps = argv[i + 1]
            i += 2
        elif argv[i] == "--env":   # NAME:K=V,K2=V2 -> an env-only variant of the default library
            name, _, kv = argv[i + 1].partition(":")
            envs[name] = dict(x.split("=", 1) for x in kv.split(",") if x)
            i += 2
        elif argv[i] == "--only":
            names = argv[i + 1].split(",")
            i += 2
        else:
            i += 1
    runs = []
    if os.path.isdir(VDIR):
        for f in sorted(os.listdir(VDIR)):
            if f.startswith("lib_") and f.endswith(".so"):
                runs.append((f[4:-3], {"OCTO_LIB": os.path.join(VDIR, f)}))
    runs += [(n, e) for n, e in envs.items()]
    for name, env in runs:
        if names and name not in names:
            continue
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", steps, "--no-e2e",
                            "--no-cpu-baseline", "--no-other-configs"], capture_output=True, text=True,
                           env=dict(os.environ, **env), timeout=900)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
            print(json.dumps({"variant": name, "value": d["value"], "ms_per_step": d["ms_per_step"],
                              "kernel_ms": d["roofline"]["kernel_ms_per_step"],
                              "clocks": d["clocks"]["sm_mhz"]}), flush=True)
        except Exception:
            print(json.dumps({"variant": name, "error": (r.stdout + r.stderr)[-1500:]}), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        run(sys.argv[2:])
