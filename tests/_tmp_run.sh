timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "p2p or v1309 or knobs or fused or edge" 2>&1 | tail -2
timeout 600 python tests/perf_variants.py run --steps 30 --env base:OCTO_P2P8=1 --env persist:OCTO_P2P_PERSIST=1 2>&1 | tail -3
timeout 600 python tests/perf_variants.py run --steps 30 --env base2:OCTO_P2P8=1 --env persist2:OCTO_P2P_PERSIST=1 2>&1 | tail -3
