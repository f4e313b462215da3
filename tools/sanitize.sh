# compute-sanitizer over the GPU parity tests (small shapes): memcheck,
# racecheck and synccheck on the attention, GEMM and model tests.
# racecheck skips the CTA-pair GEMM: its only reports are the two CTAs'
# tcgen05.alloc.cta_group::2 hardware writes of the TMEM address (ordered by
# the cluster barrier), which the tool does not model.
O=gpurun_out
T="tests/test_gpu_attention.py tests/test_gpu_gemm.py"
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest $T tests/test_gpu_model.py -q > $O/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/san_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest $T -q -k "not pair" > $O/san_racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/san_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest $T -q > $O/san_synccheck.log 2>&1; echo "synccheck rc=$?" >> $O/san_synccheck.log
for f in $O/san_*.log; do echo "== $f"; tail -4 $f; done
