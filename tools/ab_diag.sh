# live marginal cost of kernel classes in the decode step (diag_skip: 1 small ops, 2 attention, 4 GEMMs)
for mix in ${MIXES:-"" "1024:0"}; do
  echo "== mix [$mix]"
  PPD_AB="base:;nosmall:diag_skip=1;noattn:diag_skip=2;nogemm:diag_skip=4" PPD_AB_MIX=$mix PPD_AB_ROUNDS=6 timeout 300 python tools/ab_step.py 2>&1 | tail -1
done
