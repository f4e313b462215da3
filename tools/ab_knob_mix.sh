# step-level A/B of GEMM knobs over decode + prefill mixes
for mix in ${MIXES:-"512:512" "1024:0"}; do
  echo "== mix [$mix]"
  PPD_AB="base:;uniform:gemm_sched=0;balanced:gemm_sched=1;pair:gemm_pair=1;single:gemm_pair=0" PPD_AB_MIX=$mix PPD_AB_ROUNDS=5 timeout 400 python tools/ab_step.py 2>&1 | tail -1
done
