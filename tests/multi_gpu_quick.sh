#!/bin/bash
# Developer script (not a test): quick multi-GPU timing of scheduling knobs on a 4-GPU box.
set -u
cd "$(dirname "$0")/.."
T=(python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1)
python -m pytest tests/test_gpu_parity.py -x -q -k "schedule or random_amr or v1309" > gpurun_out/r2_par14.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/r2_par14.log
OCTO_M2L_SPLIT=2 OCTO_MP_BOOT=gloo OCTO_MP_TREES=amr,v1309-13 OCTO_MP_SHARDED=0 timeout 900 "${T[@]}" --nproc-per-node 4 --master-port 29651 tests/mp_fmm_run.py > gpurun_out/r2_mp4_split.log 2>&1; echo "mp4 split rc $?"; grep -a "BITWISE" gpurun_out/r2_mp4_split.log
B=(bench.py --steps 50 --no-cpu-baseline --no-other-configs --no-e2e --rank-detail)
run() { local tag=$1; shift; local n=$1; shift
  if [ $n = 1 ]; then env "$@" python "${B[@]}" > gpurun_out/r2_b14_$tag.json 2> gpurun_out/r2_b14_$tag.err
  else env "$@" "${T[@]}" --nproc-per-node $n --master-port $((29660 + RANDOM % 100)) "${B[@]}" --gpus $n > gpurun_out/r2_b14_$tag.json 2> gpurun_out/r2_b14_$tag.err; fi
  python -c "
import json; d=json.loads(open('gpurun_out/r2_b14_$tag.json').read().strip().splitlines()[-1])
print('$tag', round(d['value']/1e9,1), 'G/s', round(d['ms_per_step'],4), 'ms', {k: round(v,4) for k,v in d['roofline']['kernel_ms_per_step'].items()}, round(d['roofline']['exchange_ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
run n1 1 OCTO_M2L_SPLIT=1
run n1s 1 OCTO_M2L_SPLIT=2
run n4 4 OCTO_M2L_SPLIT=1
run n4s 4 OCTO_M2L_SPLIT=2
run n2s 2 OCTO_M2L_SPLIT=2
