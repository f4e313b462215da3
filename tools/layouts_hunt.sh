for kn in "" "mlp_fused=0" "attn_fused=0"; do
  echo "== knobs [$kn]"
  PPD_LAYOUT_KNOBS=$kn PPD_LAYOUT_QPS=6 PPD_LAYOUT_DUR=3 PPD_LAYOUT_KV=2200 PPD_LAYOUTS=4P_4D,4P_4D,4P_4D timeout 900 python tools/layouts_1gpu.py 2>&1 | grep -o '"error": "[^"]*"\|ttft_t2_p50_reduction": [0-9.]*'
done
