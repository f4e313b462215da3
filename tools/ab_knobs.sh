# A/B tuning knobs on the prefill sweep: bash tools/ab_knobs.sh "knobsA" "knobsB" ...
for r in 1 2; do
for k in "$@"; do
  PPD_PF_KNOBS=$k timeout 200 python tools/prefill_sweep.py > gpurun_out/pfk.log 2>&1
  echo "== [$k] $r"; python -c "
import json
for l in open('gpurun_out/pfk.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['m'],d['ctx'],'step',round(d['step_ms'],1),'attn',round(d['attn_ms'],2),'gemm',round(d['gemm_ms'],2),'other',round(d['step_ms']-d['attn_ms']-d['gemm_ms'],2), round(d['gemm_tflops'] or 0))
"
done; done
