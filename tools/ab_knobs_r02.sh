# knob re-check after the L2 evict-first change: L2 weight prefetch ahead of the PDL wait and PDL overlap
O=gpurun_out
for B in 16 64 200; do
  echo "== B=$B" >> $O/ab_knobs_r02.log
  PPD_AB="base:;pre16:gemm_l2_pre=16;ovl:pdl_overlap=1;both:gemm_l2_pre=16,pdl_overlap=1" PPD_AB_B=$B PPD_AB_ROUNDS=10 timeout 300 python tools/ab_step.py >> $O/ab_knobs_r02.log 2>&1
done
echo "== B=200 mix [128:896]" >> $O/ab_knobs_r02.log
PPD_AB="base:;pre16:gemm_l2_pre=16;ovl:pdl_overlap=1;both:gemm_l2_pre=16,pdl_overlap=1" PPD_AB_MIX=128:896 PPD_AB_ROUNDS=8 timeout 300 python tools/ab_step.py >> $O/ab_knobs_r02.log 2>&1
