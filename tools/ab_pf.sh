
timeout 300 python -m pytest tests/test_gpu_attention.py tests/test_gpu_model.py tests/test_gpu_engine.py -x -q > gpurun_out/pf_tests.log 2>&1
tail -3 gpurun_out/pf_tests.log
for r in 1 2; do
for v in prev cur; do
  if [ $v = cur ]; then L=paper_2603_13358_b200/libppd_b200.so; else L=ab_build/$v/paper_2603_13358_b200/libppd_b200.so; fi
  PPD_LIB=$L timeout 200 python tools/prefill_sweep.py > gpurun_out/pf_$v.$r.log 2>&1
  echo "== $v $r"; python -c "
import json,sys
for l in open('gpurun_out/pf_$v.$r.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['m'],d['ctx'],round(d['attn_ms'],2),round(d['attn_tflops'] or 0,1),round(d['step_ms'],1))
"
done
done
