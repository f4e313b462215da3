# working tree vs a baseline build (ab_build/base): decode steps and mixed decode + append steps,
# then the GPU suite and one bench line. Outputs in gpurun_out/.
O=gpurun_out
BASE=ab_build/base/paper_2603_13358_b200/libppd_b200.so
for B in 16 64 200; do
  echo "== B=$B" >> $O/ab_round.log
  PPD_AB="new:;old:@$BASE" PPD_AB_B=$B PPD_AB_ROUNDS=12 timeout 300 python tools/ab_step.py >> $O/ab_round.log 2>&1
done
for mix in "128:896" "256:768" "1536:2048"; do
  echo "== B=200 mix [$mix]" >> $O/ab_round.log
  PPD_AB="new:;old:@$BASE" PPD_AB_MIX=$mix PPD_AB_ROUNDS=10 timeout 300 python tools/ab_step.py >> $O/ab_round.log 2>&1
done
echo "== B=9 mix [1536:2048]" >> $O/ab_round.log
PPD_AB="new:;old:@$BASE" PPD_AB_B=9 PPD_AB_MIX=1536:2048 PPD_AB_ROUNDS=10 timeout 300 python tools/ab_step.py >> $O/ab_round.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests_round.log 2>&1
timeout 600 python bench.py > $O/bench_round.log 2>&1
