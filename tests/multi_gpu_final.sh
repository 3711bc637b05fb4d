#!/bin/bash
# Developer script (not a test): final multi-GPU evidence on a 4-GPU box (gpurun --gpus 4):
# bitwise multi-rank checks, configs[3] strong scaling, configs[4] weak scaling.
set -u
cd "$(dirname "$0")/.."
T=(python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1)
OCTO_MP_BOOT=gloo OCTO_MP_STEPS=4 timeout 1500 "${T[@]}" --nproc-per-node 8 --master-port 29711 tests/mp_fmm_run.py \
    > gpurun_out/r2f_mp8_gloo.log 2>&1; echo "mp8 gloo rc $?"; grep -a "BITWISE" gpurun_out/r2f_mp8_gloo.log
OCTO_MP_STEPS=4 timeout 1200 "${T[@]}" --nproc-per-node 4 --master-port 29713 tests/mp_fmm_run.py \
    > gpurun_out/r2f_mp4.log 2>&1; echo "mp4 rc $?"; grep -a "BITWISE" gpurun_out/r2f_mp4.log
B=(bench.py --steps 50 --no-cpu-baseline --no-other-configs --rank-detail)
C=(bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --rank-detail)
timeout 600 python "${B[@]}" > gpurun_out/r2f_n1.json 2> gpurun_out/r2f_n1.err
for N in 2 4; do timeout 600 "${T[@]}" --nproc-per-node $N --master-port 2972$N "${B[@]}" --gpus $N > gpurun_out/r2f_n$N.json 2> gpurun_out/r2f_n$N.err; done
timeout 1200 python "${C[@]}" > gpurun_out/r2f_c4_n1.json 2> gpurun_out/r2f_c4_n1.err
for N in 2 4; do timeout 1200 "${T[@]}" --nproc-per-node $N --master-port 2973$N "${C[@]}" --gpus $N > gpurun_out/r2f_c4_n$N.json 2> gpurun_out/r2f_c4_n$N.err; done
for f in n1 n2 n4 c4_n1 c4_n2 c4_n4; do python -c "
import json; d=json.loads(open('gpurun_out/r2f_$f.json').read().strip().splitlines()[-1])
print('$f', round(d['value']/1e9,1), 'G/s', round(d['ms_per_step'],3), 'ms', {k: round(v,3) for k,v in d['roofline']['kernel_ms_per_step'].items()}, round(d['roofline']['exchange_ms_per_step'],3), 'e2e', (d['e2e'] or {}).get('value'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
