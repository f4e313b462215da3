# mixed-step GEMM plan A/B: auto (uniform splits for 257-512 rows) vs forced balanced
# (whole waves + stream-K tail); L2 hint re-check on a prefill-heavy mix
O=gpurun_out
timeout 500 python -m pytest tests/test_gpu_model.py tests/test_gpu_attention.py tests/test_gpu_gemm.py -x -q > $O/ab_sched_tests.log 2>&1
PPD_MIX_T="200,328,456" timeout 300 python tools/gemm_mixed.py > $O/gemm_mixed_auto.log 2>&1
PPD_MIX_T="200,328,456" PPD_MIX_KNOBS="gemm_sched=1" timeout 300 python tools/gemm_mixed.py > $O/gemm_mixed_bal.log 2>&1
for mix in "128:896" "256:768"; do
  echo "== B=200 mix [$mix]" >> $O/ab_sched.log
  PPD_AB="auto:;bal:gemm_sched=1" PPD_AB_MIX=$mix PPD_AB_ROUNDS=8 timeout 300 python tools/ab_step.py >> $O/ab_sched.log 2>&1
done
echo "== B=200 mix [1536:2048] hint" >> $O/ab_sched.log
PPD_AB="h3:;h0:l2_hint=0" PPD_AB_MIX=1536:2048 PPD_AB_ROUNDS=8 timeout 300 python tools/ab_step.py >> $O/ab_sched.log 2>&1
