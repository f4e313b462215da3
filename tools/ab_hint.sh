# L2 evict-first hint A/B (knob l2_hint: bit 0 GEMM weights, bit 1 decode K/V), in-process, one build
O=gpurun_out
for B in 16 64 200; do
  echo "== B=$B" >> $O/ab_hint2.log
  PPD_AB="h3:l2_hint=3;h2:l2_hint=2;h1:l2_hint=1;h0:l2_hint=0" PPD_AB_B=$B PPD_AB_ROUNDS=12 timeout 300 python tools/ab_step.py >> $O/ab_hint2.log 2>&1
done
for mix in "128:896" "1536:2048"; do
  echo "== B=200 mix [$mix]" >> $O/ab_hint2.log
  PPD_AB="h3:l2_hint=3;h2:l2_hint=2;h1:l2_hint=1;h0:l2_hint=0" PPD_AB_MIX=$mix PPD_AB_ROUNDS=8 timeout 300 python tools/ab_step.py >> $O/ab_hint2.log 2>&1
done
echo "== B=16 mix [1536:2048]" >> $O/ab_hint2.log
PPD_AB="h3:l2_hint=3;h2:l2_hint=2;h0:l2_hint=0" PPD_AB_B=16 PPD_AB_MIX=1536:2048 PPD_AB_ROUNDS=8 timeout 300 python tools/ab_step.py >> $O/ab_hint2.log 2>&1
