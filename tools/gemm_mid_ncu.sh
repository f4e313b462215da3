# prefill-size GEMM evidence: the tcgen05 vs cuBLAS table, then one ncu --set full
# capture of the fused gate|up GEMM at T=1736 and of the down GEMM at T=4096
O=gpurun_out
timeout 300 python tools/gemm_mid.py > $O/gemm_mid.log 2>&1; cat $O/gemm_mid.log
PPD_ONE="1736:28672:4096:0:-1" timeout 300 ncu --set full --clock-control none -k regex:gemm_tc -s 1 -c 1 -o $O/gemm_gu1736 python tools/gemm_one.py > $O/gemm_ncu1.log 2>&1
PPD_ONE="4096:4096:14336:1:-1" timeout 300 ncu --set full --clock-control none -k regex:gemm_tc -s 1 -c 1 -o $O/gemm_down4096 python tools/gemm_one.py > $O/gemm_ncu2.log 2>&1
tail -2 $O/gemm_ncu1.log $O/gemm_ncu2.log
