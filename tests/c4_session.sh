#!/bin/bash
# Developer script (not a test): configs[4] (V1309 level 15 + common envelope, weak scaling,
# ~1.2 M level-15 sub-grids per GPU) at N = 1, 2, 4 on a 4-GPU box.
set -u
cd "$(dirname "$0")/.."
T=(python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1)
B=(bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --rank-detail)
timeout 1500 python "${B[@]}" > gpurun_out/r2_c4_n1.json 2> gpurun_out/r2_c4_n1.err; echo "c4 n1 rc $?"
for N in 2 4; do
  timeout 1500 "${T[@]}" --nproc-per-node $N --master-port 2967$N "${B[@]}" --gpus $N > gpurun_out/r2_c4_n$N.json 2> gpurun_out/r2_c4_n$N.err
  echo "c4 n$N rc $?"
done
for N in 1 2 4; do python -c "
import json; d=json.loads(open('gpurun_out/r2_c4_n$N.json').read().strip().splitlines()[-1])
print('c4 n$N', round(d['value']/1e9,1), 'G/s', round(d['ms_per_step'],2), 'ms', d['config']['subgrids'], {k: round(v,3) for k,v in d['roofline']['kernel_ms_per_step'].items()}, round(d['roofline']['exchange_ms_per_step'],3), d['config']['hbm_used_gb_rank0'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
