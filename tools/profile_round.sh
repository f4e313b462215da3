#!/bin/bash
# One gpurun call's worth of round evidence: the headline bench line, the ncu
# launch list of one decode step, ncu --set full of the step's top kernels
# and of the K2 mixed launch, and the GPU test suite. Outputs in gpurun_out/.
#   gpurun --timeout 1500 -- 'bash tools/profile_round.sh TAG'
TAG=${1:-r01}
O=gpurun_out
timeout 600 python bench.py > $O/bench_$TAG.log 2>&1
PPD_NCU=1 timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/launches_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --fill-kv random --no-cpu --no-engine > $O/ncu_launch_$TAG.log 2>&1
PPD_NCU=1 timeout 400 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:"decode_attention|gemm_tc" -c 6 -o $O/step_full_$TAG \
  python bench.py --steps 1 --warmup 1 --fill-kv random --no-cpu --no-engine > $O/ncu_full_$TAG.log 2>&1
PPD_AB=fused: PPD_AB_MIX=128:896 PPD_AB_ROUNDS=1 PPD_AB_STEPS=1 timeout 300 ncu --set full --import-source on \
  --clock-control none -k regex:mixed_attention -s 40 -c 1 -o $O/mixed_full_$TAG \
  python tools/ab_step.py > $O/ncu_mixed_$TAG.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > $O/gpu_tests_$TAG.log 2>&1
echo done > $O/profile_$TAG.done
