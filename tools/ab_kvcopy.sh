for r in 1 2; do
echo "== prev"; PPD_LIB=ab_build/prev/paper_2603_13358_b200/libppd_b200.so timeout 200 python tools/kv_copy_bench.py 2>&1 | tail -4
echo "== cur"; timeout 200 python tools/kv_copy_bench.py 2>&1 | tail -4
done
timeout 300 python -m pytest tests/test_gpu_model.py tests/test_gpu_engine.py -x -q 2>&1 | tail -1
