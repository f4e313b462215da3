# compute-sanitizer over the GPU parity tests (tiny shapes): memcheck on the
# attention / model / engine tests, racecheck + synccheck on the attention tests.
O=gpurun_out
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_attention.py tests/test_gpu_model.py -x -q > $O/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/san_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_attention.py -x -q -k "full_prefill or append_prefill or mixed_decode" > $O/san_racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/san_racecheck.log
timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_attention.py -x -q -k "full_prefill or append_prefill or mixed_decode" > $O/san_synccheck.log 2>&1; echo "synccheck rc=$?" >> $O/san_synccheck.log
tail -3 $O/san_*.log
