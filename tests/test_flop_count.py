"""bench.py's per-interaction flop constants (the roofline numerator, C10)
equal the op counts of the shipped kernels' inner loops (tests/flop_count.py,
from the SASS of libocto_fmm.so).  CPU-only: cuobjdump reads the sm_100a
binary without a GPU."""
import os
import shutil
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump not installed")
def test_bench_flops_equal_sass_counts():
    import flop_count
    import paper_1908_03121_b200 as P
    P.lib()   # builds the library if the sources are newer
    import bench
    got = {k: v["flop"] for k, v in flop_count.derive().items()}
    assert got == bench.FLOPS, (got, bench.FLOPS)
