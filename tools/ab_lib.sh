# step-level A/B of the working tree against another build: bash tools/ab_lib.sh ab_build/<name> [mixes...]
OLD=$1; shift
timeout 400 python -m pytest tests/test_gpu_model.py tests/test_gpu_attention.py -x -q 2>&1 | tail -2
for mix in "$@"; do
  echo "== mix [$mix]"
  PPD_AB="new:;old:@$OLD/paper_2603_13358_b200/libppd_b200.so" PPD_AB_MIX=$mix PPD_AB_ROUNDS=8 timeout 300 python tools/ab_step.py 2>&1 | tail -1
done
