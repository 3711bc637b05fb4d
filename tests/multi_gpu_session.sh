#!/bin/bash
# Developer script (not a test): the multi-GPU evidence run on a 4-GPU box
# (gpurun --gpus 4).  Writes logs / JSON lines under gpurun_out/ for profiles/.
#   1. 8 ranks on 4 GPUs (2 per GPU), one-sided exchange bootstrapped over gloo: bitwise vs 1 rank
#   2. 4 ranks, one per GPU, library NCCL bootstrap, one-sided puts: bitwise vs 1 rank
#   3. bench.py strong scaling on configs[3] at N = 1, 2, 4 (+ N = 4 with the leaf kernels beside M2L)
set -u
cd "$(dirname "$0")/.."
T=(python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1)
OCTO_MP_BOOT=gloo OCTO_MP_STEPS=4 timeout 1500 "${T[@]}" --nproc-per-node 8 --master-port 29611 tests/mp_fmm_run.py \
    > gpurun_out/r2_mp8_gloo.log 2>&1; echo "mp8 gloo rc $?"; grep -a "BITWISE\|MISMATCH" gpurun_out/r2_mp8_gloo.log | head -5
OCTO_MP_STEPS=4 timeout 1200 "${T[@]}" --nproc-per-node 4 --master-port 29613 tests/mp_fmm_run.py \
    > gpurun_out/r2_mp4_puts.log 2>&1; echo "mp4 puts rc $?"; grep -a "BITWISE\|MISMATCH" gpurun_out/r2_mp4_puts.log | head -5
B=(bench.py --steps 50 --no-cpu-baseline --no-other-configs --rank-detail)
timeout 600 python "${B[@]}" > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench_n1.err; echo "n1 rc $?"
for N in 2 4; do
  timeout 600 "${T[@]}" --nproc-per-node $N --master-port 2962$N "${B[@]}" --gpus $N > gpurun_out/r2_bench_n$N.json 2> gpurun_out/r2_bench_n$N.err
  echo "n$N rc $?"
done
OCTO_CONCURRENCY=1 timeout 600 "${T[@]}" --nproc-per-node 4 --master-port 29631 "${B[@]}" --gpus 4 \
    > gpurun_out/r2_bench_n4_conc.json 2> gpurun_out/r2_bench_n4_conc.err; echo "n4 conc rc $?"
for f in n1 n2 n4 n4_conc; do python -c "
import json,sys; d=json.load(open('gpurun_out/r2_bench_$f.json'))
print('$f', round(d['value']/1e9,1), 'G/s', round(d['ms_per_step'],3), 'ms', d['roofline']['kernel_ms_per_step'], 'x', round(d['roofline']['exchange_ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e9,1), d['clocks'])"; done
