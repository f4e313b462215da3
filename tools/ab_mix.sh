for mix in "" "128:896" "512:512" "1024:0" "1536:2048"; do
  echo "== mix [$mix]"
  PPD_AB="never:mlp_fused=0;always:mlp_fused=1" PPD_AB_MIX=$mix PPD_AB_ROUNDS=6 timeout 300 python tools/ab_step.py 2>&1 | tail -3
done
